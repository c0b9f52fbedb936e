"""Small end-to-end run of every C-ABI entry point (LCP-hist, accumulate, DP int32/int64/fp64
including the task-pool and small-N paths, evaluation) for compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_05219_b200 import sp
from paper_2605_05219_b200 import workload as wl

dev = torch.device("cuda:0")
# LCP + histogram (aligned and scalar paths)
for align in (4, 1):
    cfg = wl.TraceConfig(**{**wl.scaled(wl.CONFIGS["W2"], 6).__dict__, "align": align})
    tr = wl.make_trace(cfg, seed=1)
    g = {k: v.to(dev) for k, v in tr.items() if isinstance(v, torch.Tensor)}
    lcp = torch.empty(g["req_off"].numel() - 1, dtype=torch.int32, device=dev)
    h, _ = sp.overlap_hist(g["entry_tokens"], g["entry_off"], g["req_tokens"], g["req_off"],
                           g["req_entry"], cfg.N, lcp_out=lcp, n_entries=6)
    sp.accumulate_depths(g["req_entry"], lcp, 0, 3, cfg.N, torch.zeros(3, cfg.N + 1, dtype=torch.int32, device=dev))
# DP: small N (top/run_level path), N >= 1024 (task pool + segments), int64 and fp64 paths
for N, M, E in ((37, 5, 9), (300, 12, 6), (2048, 8, 4), (5000, 16, 3)):
    cfg = wl.TraceConfig("s", E, N, M, 1, (N, N), (1, 1), "mix", dense_n=(N // 2, 2 * N))
    H = wl.make_dense_hist(cfg, seed=N).to(dev)
    sp.place_checkpoints(H, M, cost_by_budget=True)
    sp.place_checkpoints(H.to(torch.int64) * 40000, M, cost_by_budget=True)
    sp.place_checkpoints(H.to(torch.float64) / H.sum(1, keepdim=True), M, cost_by_budget=True)
    pos, npos, _ = sp.baseline_sets(N, budgets=(1, M), blocks=(64,), device=dev)
    sp.expected_recompute(H, pos, npos)
    sp.expected_recompute(H.to(torch.float64), pos, npos)
torch.cuda.synchronize()
print("sanitize_small ok")
