"""Seeded synthetic query-graph generators shared by the tests, bench.py and the
oracle harness.  This module holds NO arithmetic of the method (no cardinality
products, no costs, no enumeration): it only draws graphs and numbers.
"""
from .gen import (QueryGraph, star, snowflake, chain, cycle, clique, random_connected,
                  fig5_fixture, fig3_fixture, generate, from_json, to_json)

__all__ = ["QueryGraph", "star", "snowflake", "chain", "cycle", "clique",
           "random_connected", "fig5_fixture", "fig3_fixture", "generate",
           "from_json", "to_json"]
