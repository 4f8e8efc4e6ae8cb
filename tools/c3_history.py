"""Checks that C3 s/decision does not depend on what the context ran before
(capacity growth from a larger search must not slow later, smaller ones)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_2207_06649_b200 import Context

ctx = Context(0)
print(json.dumps({"c3_fresh": bench.c3_episodes(ctx, False)}), flush=True)
print(json.dumps({"c3_again": bench.c3_episodes(ctx, False)}), flush=True)
print(json.dumps({"c4": bench.c4_decision(ctx, False)}), flush=True)
print(json.dumps({"c3_after_c4": bench.c3_episodes(ctx, False)}), flush=True)
