"""The fp64 (a7) step's pieces on W5-shaped rows, timed one by one with CUDA events: the DP with
and without V_0..V_M (cost_by_budget: the definitional cost of every budget's canonical
placement, reading R10), on w = c / n and on unnormalised rows W = c, and the fp64 evaluation of
the Table 1 baselines."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_05219_b200 import sp
from paper_2605_05219_b200 import workload as wl

ap = argparse.ArgumentParser()
ap.add_argument("--entries", type=int, default=16384)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
cfg = wl.scaled(wl.CONFIGS["W5"], a.entries)
dev = torch.device("cuda:0")
H = wl.make_dense_hist(cfg, seed=0, device=dev)
Wn = (H.double() / H.sum(1, keepdim=True).double()).contiguous()
Wc = H.double().contiguous()
del H
E, N, M = a.entries, cfg.N, cfg.M
ws = torch.empty(sp.place_checkpoints_workspace_bytes(E, N, M), dtype=torch.uint8, device=dev)
bpos, bnpos, _ = sp.baseline_sets(N, budgets=(M,), blocks=(64, 128), device=dev)


def timed(fn):
    for r in range(a.reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
    return s.elapsed_time(e)


for name, W in (("w=c/n", Wn), ("W=c", Wc)):
    t0 = timed(lambda: sp.place_checkpoints(W, M, workspace=ws))
    t1 = timed(lambda: sp.place_checkpoints(W, M, cost_by_budget=True, workspace=ws))
    t2 = timed(lambda: sp.expected_recompute(W, bpos, bnpos))
    st = sp.dp_stats(ws)
    print(f"{name}: dp {t0:.3f} ms, dp + V_0..V_M {t1:.3f} ms, eval {t2:.3f} ms; "
          f"hull={st['entries_hull']} f64={st['entries_f64']} evals={st['evaluations']}", flush=True)
