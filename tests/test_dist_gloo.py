"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: request routing, padding, the
all-gather / all-reduce exchange and owner slicing in paper_2605_05219_b200.dist.  The device
kernels are replaced by CPU stand-ins with the same contract (the depth of a request is the
generator's drawn depth clamped to N, which the GPU parity tests pin for the LCP kernel); the
merged per-owner histograms must equal a single-process histogram of all requests."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_05219_b200 import workload as wl


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def cpu_accumulate(entry, depth, e_begin, e_end, N, hist, stream=None):
    """CPU stand-in for sp_accumulate_depths (same documented contract)."""
    e = entry.numpy().astype(np.int64)
    d = depth.numpy().astype(np.int64)
    m = (e >= e_begin) & (e < e_end) & (d >= 0) & (d <= N)
    h = hist.numpy()
    np.add.at(h, (e[m] - e_begin, d[m]), 1)
    return hist


def _worker(rank, world, port, mode, E_own, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_05219_b200.dist import HistMerger
    cfg = wl.scaled(wl.CONFIGS["W2"], E_own * world)
    cfg = wl.TraceConfig(**{**cfg.__dict__, "N": 700})
    tr = wl.make_trace(cfg, seed=5, world=world, rank=rank)
    N = cfg.N
    merger = HistMerger(tr["req_entry"], E_own, N, mode=mode, accumulate=cpu_accumulate)
    depth = torch.clamp(tr["depth"], max=N)
    R = depth.numel()
    hist_own = torch.zeros(E_own, N + 1, dtype=torch.int32)
    for step in range(2):                      # two steps: buffers are reusable
        if mode == "sparse":
            merger.lcp_out[:R] = depth         # what sp_overlap_hist(lcp_out=...) writes
        else:
            np.add.at(merger.partial.numpy(), (tr["req_entry"].numpy(), depth.numpy()), 1)
        merger.merge(hist_own)
    gathered = [torch.zeros_like(hist_own) for _ in range(world)]
    dist.all_gather(gathered, hist_own)
    counts = torch.tensor([R])
    allc = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(allc, counts)
    if rank == 0:
        out.put((torch.cat(gathered).numpy(), [int(c) for c in allc]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["sparse", "allreduce"])
def test_two_rank_merge_equals_single_process(mode):
    world, E_own = 2, 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, E_own, q))
             for r in range(world)]
    for p in procs:
        p.start()
    merged, counts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference: every request of every entry, once per step (2 steps)
    cfg = wl.scaled(wl.CONFIGS["W2"], E_own * world)
    cfg = wl.TraceConfig(**{**cfg.__dict__, "N": 700})
    tr = wl.make_trace(cfg, seed=5)
    ref = np.zeros((E_own * world, cfg.N + 1), np.int64)
    np.add.at(ref, (tr["req_entry"].numpy(), np.minimum(tr["depth"].numpy(), cfg.N)), 2)
    assert sum(counts) == tr["req_entry"].numel()        # routing is a partition
    assert min(counts) > 0
    assert (merged == ref).all()


def test_routing_partitions_requests():
    cfg = wl.scaled(wl.CONFIGS["W3"], 6)
    full = wl.make_trace(cfg, seed=2)
    parts = [wl.make_trace(cfg, seed=2, world=3, rank=r) for r in range(3)]
    assert sum(p["req_entry"].numel() for p in parts) == full["req_entry"].numel()
    # same multiset of (entry, depth) and identical entry tokens on every rank
    key = lambda t: sorted(zip(t["req_entry"].tolist(), t["depth"].tolist()))  # noqa: E731
    allp = sorted(sum((list(zip(p["req_entry"].tolist(), p["depth"].tolist())) for p in parts), []))
    assert allp == key(full)
    for p in parts:
        assert torch.equal(p["entry_tokens"], full["entry_tokens"])
