"""Profiling driver: one warm-up + one measured sp_place_checkpoints launch on W5-shaped dense
histograms (E entries), then the LCP kernel on a W5-shaped trace.  Used under ncu."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_05219_b200 import sp
from paper_2605_05219_b200 import workload as wl

ap = argparse.ArgumentParser()
ap.add_argument("--entries", type=int, default=148)
ap.add_argument("--workload", default="W5")
ap.add_argument("--M", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--lcp", action="store_true")
ap.add_argument("--plus1", action="store_true", help="add 1 to every bin (full support, K = N)")
ap.add_argument("--ones", action="store_true", help="all-ones rows (the large-hull mode)")
ap.add_argument("--dense-n", type=int, nargs=2, default=None, help="draws per entry (lo hi)")
ap.add_argument("--no-hull", action="store_true", help="D&C kernel only (SP_NO_HULL)")
ap.add_argument("--f64", action="store_true", help="fp64 weights w = c / n (a7)")
ap.add_argument("--sort-support", action="store_true", help="rows permuted by support, largest first")
a = ap.parse_args()
cfg = wl.scaled(wl.CONFIGS[a.workload], a.entries)
if a.dense_n:
    import dataclasses
    cfg = dataclasses.replace(cfg, dense_n=tuple(a.dense_n))
if a.no_hull:
    os.environ["SP_NO_HULL"] = "1"
M = a.M or cfg.M
dev = torch.device("cuda:0")
H = wl.make_dense_hist(cfg, seed=0, device=dev) if cfg.dense_n and not a.ones else wl.uniform_hist(a.entries, cfg.N, dev)
if a.plus1:
    H[:, 1:] += 1
if a.sort_support:
    H = H[torch.argsort((H[:, 1:] > 0).sum(1), descending=True)].contiguous()
if a.f64:
    H = (H.double() / H.sum(1, keepdim=True).double()).contiguous()
ws = torch.empty(sp.place_checkpoints_workspace_bytes(a.entries, cfg.N, M), dtype=torch.uint8, device=dev)
for r in range(a.reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    sp.place_checkpoints(H, M, workspace=ws)
    e.record()
    torch.cuda.synchronize()
    st = sp.dp_stats(ws)
    print(f"dp rep {r}: {s.elapsed_time(e):.3f} ms  cells={a.entries*cfg.N*M:.3e} "
          f"evals/cell={st['evaluations']/(a.entries*cfg.N*M):.2f}  "
          f"Mcells/s={a.entries*cfg.N*M/s.elapsed_time(e)/1e3:.1f}  "
          f"hull={st['entries_hull']} big={st['entries_hull_big']} support_rows/entry={st['hull_event_rows']/max(1,st['entries_hull']):.0f} "
          f"pops/support-cell={st['hull_pops']/max(1,st['hull_event_rows']*M):.3f}", flush=True)
if os.environ.get("SP_TAIL_REPORT"):   # needs SP_NVCC_EXTRA=-DSP_HULL_TAIL; last rep
    v = ws[:128].view(torch.int64).cpu().tolist()
    end, nstart, busy, nw = v[11], v[12], v[13], v[14]
    span = end - (2**64 - 1 - (nstart & (2**64 - 1)))   # t_start = ~(stored complement)
    print(f"tail: {nw} warps, span {span/1e6:.3f} ms, mean warp busy {busy/max(nw,1)/1e6:.3f} ms, "
          f"utilisation {busy/max(nw,1)/max(span,1):.3f}")
if a.lcp:
    tr = wl.make_trace(cfg, seed=0, device=dev)
    lcp = torch.empty(tr["req_off"].numel() - 1, dtype=torch.int32, device=dev)
    hist = torch.zeros(a.entries, cfg.N + 1, dtype=torch.int32, device=dev)
    for r in range(a.reps):
        sp.overlap_hist(tr["entry_tokens"], tr["entry_off"], tr["req_tokens"], tr["req_off"],
                        tr["req_entry"], cfg.N, hist=hist, lcp_out=lcp)
    torch.cuda.synchronize()
if os.environ.get("SP_TIMING_REPORT"):
    v = ws[:128].view(torch.int64).cpu().tolist()
    names = ["rowN", "top", "segments(+barrier)", "reload", "seg warp busy (sum)", "seg max-warp busy (sum)", "seg passes (warp sum)", "seg long rows (warp sum)"]
    tot = sum(v[8:12])
    for i, nm in enumerate(names[:8]):
        print(f"  {nm:28s} {v[8+i]/1e6:10.2f} Mcyc  ({v[8+i]/max(tot,1)*100:5.1f}% of phase total)" if i < 4 else f"  {nm:28s} {v[8+i]/1e6:10.2f} Mcyc")
    nw = 32
    print(f"  segment phase: mean warp busy / max warp busy = {v[12]/nw/max(v[13],1):.2f}")
if os.environ.get("SP_BRSTATS_REPORT"):
    v = ws[:128].view(torch.int64).cpu().tolist()
    print(f"brstats: support rows (warp-steps) {v[8]}, back-pop loop taken {v[9]} ({v[9]/max(v[8],1)*100:.1f}%), "
          f"front-pop loop taken {v[10]} ({v[10]/max(v[8],1)*100:.1f}%)  [counts summed over {a.reps} reps]")
