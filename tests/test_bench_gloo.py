"""World-size-2 gloo test (CPU) of bench.py's N > 1 step path (HotPath): request routing,
strong-scaling entry ownership, the sparse and the dense merge, and the per-owner DP and
baseline evaluation.  The device kernels are replaced by CPU stand-ins built on the oracle (the
GPU parity tests pin the kernels against the same oracle); every owner's placements, costs,
V_0..V_M and baseline costs must equal a single-process run over all requests (integer sums
commute: SURVEY 8(c) row e)."""
import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import oracle
from paper_2605_05219_b200 import sp
from paper_2605_05219_b200 import workload as wl


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cpu_ops():
    """CPU stand-ins with the device calls' contracts (sp.overlap_hist, sp.accumulate_depths,
    sp.place_checkpoints, sp.expected_recompute)."""
    def overlap_hist(entry_tokens, entry_off, req_tokens, req_off, req_entry, N, hist=None,
                     lcp_out=None, n_entries=None, stream=None, with_hist=True):
        h, l = oracle.lcp_hist(entry_tokens.numpy(), entry_off.numpy(), req_tokens.numpy(),
                               req_off.numpy(), req_entry.numpy(), N, n_entries=n_entries)
        if with_hist and hist is not None:
            hist += torch.from_numpy(h.astype(np.int32))
        if lcp_out is not None:
            lcp_out[:l.size] = torch.from_numpy(l.astype(np.int32))
        return hist, lcp_out

    def accumulate_depths(entry, depth, e_begin, e_end, N, hist, stream=None):
        e = entry.numpy().astype(np.int64)
        d = depth.numpy().astype(np.int64)
        m = (e >= e_begin) & (e < e_end) & (d >= 0) & (d <= N)
        np.add.at(hist.numpy(), (e[m] - e_begin, d[m]), 1)
        return hist

    def place_checkpoints(w, M, positions=None, n_positions=None, cost=None,
                          cost_by_budget=None, workspace=None, stream=None):
        p, k, c, cb = oracle.place_batch(w.numpy(), M, "cht", with_budget=True)
        positions.copy_(torch.from_numpy(p))
        n_positions.copy_(torch.from_numpy(k))
        cost.copy_(torch.from_numpy(c))
        cost_by_budget.copy_(torch.from_numpy(cb))

    def expected_recompute(w, pos, npos, broadcast=True, cost=None, worst=None, stream=None):
        c, wc = oracle.eval_batch(w.numpy(), pos.numpy(), npos.numpy(), broadcast=broadcast)
        cost.copy_(torch.from_numpy(c))
        worst.copy_(torch.from_numpy(wc))

    return types.SimpleNamespace(
        overlap_hist=overlap_hist, accumulate_depths=accumulate_depths,
        place_checkpoints=place_checkpoints, expected_recompute=expected_recompute,
        place_checkpoints_workspace_bytes=lambda E, N, M: 0, baseline_sets=sp.baseline_sets)


def _cfg():
    c = wl.scaled(wl.CONFIGS["W2"], 8)
    return wl.TraceConfig(**{**c.__dict__, "N": 300, "L_range": (150, 300), "M": 6})


def _run(world, rank, merge, steps=2):
    args = types.SimpleNamespace(scaling="strong", entries=8)
    E_tot, E_own = bench.plan_entries(args, _cfg(), world)
    hp = bench.HotPath(_cfg(), E_tot, E_own, world, rank, merge, 3, "cpu", ops=_cpu_ops())
    for _ in range(steps):
        hp.step()
    return [t.clone() for t in (hp.hist, hp.positions, hp.npos, hp.cost, hp.cbb, hp.bcost,
                                hp.bworst)]


def _worker(rank, world, port, merge, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = _run(world, rank, merge)
    gathered = []
    for t in res:
        g = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(g, t)
        gathered.append(torch.cat(g).numpy())
    if rank == 0:
        out.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("merge", ["sparse", "allreduce"])
def test_bench_step_world2_equals_single_process(merge):
    assert "L_range" in wl.TraceConfig.__dataclass_fields__
    ref = [t.numpy() for t in _run(1, 0, merge)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, merge, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    names = ["hist", "positions", "npos", "cost", "cbb", "bcost", "bworst"]
    for name, a, b in zip(names, got, ref):
        assert a.shape == b.shape and (a == b).all(), name
    assert ref[0].sum() > 0 and (ref[2] > 0).any()


def test_plan_entries_strong_and_weak():
    cfg = wl.CONFIGS["W5"]
    s = types.SimpleNamespace(scaling="strong", entries=None)
    assert bench.plan_entries(s, cfg, 8) == (16384, 2048)
    assert bench.plan_entries(s, cfg, 1) == (16384, 16384)
    w = types.SimpleNamespace(scaling="weak", entries=None)
    assert bench.plan_entries(w, cfg, 8) == (131072, 16384)
