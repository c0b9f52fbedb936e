"""Experiment: overlap the HBM-bound LCP kernel with the ALU-bound hull DP across entry blocks.

Serial step (bench.py): LCP(all) -> DP(all) -> eval(all) on one stream.  Overlapped step: the
entries are cut into C blocks (requests are grouped by entry, so a block's requests are
contiguous); the LCP of block c runs on the main stream, and block c's DP + evaluation run on
one of two side streams (own workspace each) once its LCP is done, so LCP(c+1) runs beside
DP(c) and each DP launch's tail is filled by the next one's warps.  Prints both step times and
checks that the two schedules give identical outputs; also times the evaluation on a side
stream beside the DP (it needs only the histograms).  W5, device-resident inputs.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_05219_b200 import sp
from paper_2605_05219_b200 import workload as wl

ap = argparse.ArgumentParser()
ap.add_argument("--chunks", type=int, nargs="+", default=[2, 4, 8])
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()

dev = torch.device("cuda:0")
cfg = wl.CONFIGS["W5"]
E, N, M = cfg.n_entries, cfg.N, cfg.M
tr = wl.make_trace(cfg, seed=0, device=dev)
hist0 = wl.make_dense_hist(cfg, seed=0, device=dev, entry_begin=0, n_entries=E)
bpos, bnpos, _ = sp.baseline_sets(N, budgets=(M,), blocks=(64, 128), device=dev)
S = bpos.shape[0]
R = tr["req_off"].numel() - 1
ent = tr["req_entry"].cpu().numpy()


def outputs():
    return dict(hist=hist0.clone(), positions=torch.empty(E, M, dtype=torch.int32, device=dev),
                npos=torch.empty(E, dtype=torch.int32, device=dev),
                cost=torch.empty(E, dtype=torch.int64, device=dev),
                cbb=torch.empty(E, M + 1, dtype=torch.int64, device=dev),
                bcost=torch.empty(E, S, dtype=torch.int64, device=dev),
                bworst=torch.empty(E, S, dtype=torch.int32, device=dev),
                lcp=torch.full((R,), -1, dtype=torch.int32, device=dev))


main = torch.cuda.current_stream(dev)
side = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
wsb = sp.place_checkpoints_workspace_bytes(E, N, M)
ws = [torch.empty(wsb, dtype=torch.uint8, device=dev) for _ in range(2)]


def lcp(o, r0, r1, st):
    if r1 > r0:
        sp.overlap_hist(tr["entry_tokens"], tr["entry_off"], tr["req_tokens"],
                        tr["req_off"][r0:r1 + 1], tr["req_entry"][r0:r1], N, hist=o["hist"],
                        lcp_out=o["lcp"][r0:r1], n_entries=E, stream=st)


def dp_eval(o, e0, e1, w, st):
    h = o["hist"][e0:e1]
    sp.place_checkpoints(h, M, positions=o["positions"][e0:e1], n_positions=o["npos"][e0:e1],
                         cost=o["cost"][e0:e1], cost_by_budget=o["cbb"][e0:e1], workspace=w,
                         stream=st)
    sp.expected_recompute(h, bpos, bnpos, broadcast=True, cost=o["bcost"][e0:e1],
                          worst=o["bworst"][e0:e1], stream=st)


def step_serial(o):
    lcp(o, 0, R, main)
    dp_eval(o, 0, E, ws[0], main)


def step_overlap(o, C):
    eb = [E * c // C for c in range(C + 1)]
    rb = [int(np.searchsorted(ent, x, side="left")) for x in eb]
    for c in range(C):
        lcp(o, rb[c], rb[c + 1], main)
        ev = torch.cuda.Event()
        ev.record(main)
        s = side[c & 1]
        s.wait_event(ev)
        dp_eval(o, eb[c], eb[c + 1], ws[c & 1], s)
    for s in side:
        main.wait_stream(s)


def step_eval_side(o):
    """The evaluation needs only the histograms: run it on a side stream beside the DP, where
    its CTAs can take the SMs the DP's tail leaves idle."""
    lcp(o, 0, R, main)
    ev = torch.cuda.Event()
    ev.record(main)
    side[0].wait_event(ev)
    sp.expected_recompute(o["hist"], bpos, bnpos, broadcast=True, cost=o["bcost"],
                          worst=o["bworst"], stream=side[0])
    sp.place_checkpoints(o["hist"], M, positions=o["positions"], n_positions=o["npos"],
                         cost=o["cost"], cost_by_budget=o["cbb"], workspace=ws[0], stream=main)
    main.wait_stream(side[0])


def timed(fn, o):
    for _ in range(a.warmup):
        o["hist"].copy_(hist0)
        fn(o)
    torch.cuda.synchronize()
    t = 0.0
    for _ in range(a.steps):      # the histogram reset is outside the timed region
        o["hist"].copy_(hist0)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record(main)
        fn(o)
        e.record(main)
        torch.cuda.synchronize()
        t += s.elapsed_time(e)
    return t / a.steps


ref = outputs()
t_ser = timed(step_serial, ref)
print(f"serial: {t_ser:.3f} ms/step", flush=True)
o = outputs()
t = timed(step_eval_side, o)
print(f"eval on a side stream beside the DP: {t:.3f} ms/step ({t_ser / t:.3f}x)  outputs identical: "
      f"{all(torch.equal(ref[k], o[k]) for k in ref)}", flush=True)
for C in a.chunks:
    o = outputs()
    t = timed(lambda x: step_overlap(x, C), o)
    same = all(torch.equal(ref[k], o[k]) for k in ref)
    print(f"overlap C={C}: {t:.3f} ms/step ({t_ser / t:.3f}x)  outputs identical: {same}",
          flush=True)
