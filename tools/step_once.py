"""One eager hot-path step at the bench workload (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse

import bench

a = bench.parse()
a.no_graph = True
a.warmup = 1
a.steps = 1
a.e2e_steps = 1
a.no_cpu_baseline = True
import torch  # noqa: E402

res = bench.run_ours(a, 0, 1, None)
print("ms", res["ms"], res["phase_ms"])
