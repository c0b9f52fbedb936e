"""Profiling driver for a6 (sp_expected_recompute) on W5-shaped dense histograms with the bench's
baseline sets (balanced M, block B = 64 and 128): times the default (broadcast-table) kernel and the
shared-prefix kernel (SP_DBG_EVAL_PATH = 3) and checks that they agree on every entry."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_05219_b200 import sp
from paper_2605_05219_b200 import workload as wl

ap = argparse.ArgumentParser()
ap.add_argument("--entries", type=int, default=16384)
ap.add_argument("--workload", default="W5")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--sweep", action="store_true", help="the workload's budget sweep (W4: M = 1..64)")
a = ap.parse_args()
cfg = wl.scaled(wl.CONFIGS[a.workload], a.entries)
dev = torch.device("cuda:0")
H = wl.make_dense_hist(cfg, seed=0, device=dev)
budgets = cfg.M_sweep if a.sweep and cfg.M_sweep else (cfg.M,)
bpos, bnpos, _ = sp.baseline_sets(cfg.N, budgets=budgets, blocks=(64, 128), device=dev)
print(f"{cfg.name}: {cfg.n_entries} entries, N={cfg.N}, {bpos.shape[0]} broadcast sets")
out = {}
for name, path in (("auto", 0), ("prefix", 3), ("chunked", 1)):
    dbg = sp.debug(SP_DBG_EVAL_PATH=path)
    dbg.__enter__()
    ts = []
    for r in range(a.reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        c, w = sp.expected_recompute(H, bpos, bnpos, broadcast=True)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    dbg.__exit__(None, None, None)
    out[name] = (c, w)
    gb = H.numel() * 4 / 1e9
    print(f"{name}: " + " ".join(f"{t:.3f}" for t in ts) + f" ms  ({gb:.2f} GB row bytes, "
          f"{gb / min(ts) * 1e3:.0f} GB/s at best)", flush=True)
print("agree:", all(bool(torch.equal(out["auto"][i], out[k][i])) for k in ("prefix", "chunked")
                    for i in (0, 1)))
