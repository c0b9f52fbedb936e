"""The one exchange step of the multi-GPU path: merging overlap-depth
observations of requests that arrived on other ranks into the owner's histograms.

Entries are sharded in contiguous blocks (rank r owns [r E_own, (r+1) E_own)); each entry's DP
is independent (per-edge decomposition), so after the merge every rank places
checkpoints for its own entries with no further communication.  Requests arrive on any rank
(workload.make_trace(world=, rank=)), and their LCP runs where they arrived (entry tokens are
replicated).  Two merge modes, identical results (integer sums commute):

  sparse    (default) all-gather of the (entry, depth) pairs -- 4 B per request, the entry ids
            gathered once per batch -- then each owner scatter-adds its own pairs with the
            sp_accumulate_depths kernel.  Traffic: 4 R_total bytes per rank and step.
  allreduce the BASELINE.json north_star's dense variant: every rank accumulates a partial
            int32 histogram over ALL entries, NCCL all-reduces it (SUM), and the owner adds its
            slice.  Traffic: ~2 E_total (N+1) 4 bytes per rank and step; kept for comparison.

torch.distributed is plumbing here (NCCL on GPU, gloo in the CPU tests); the arithmetic of the
merge runs in the library's kernels (sp_overlap_hist / sp_accumulate_depths).
"""
from __future__ import annotations

import contextlib

import torch
import torch.distributed as dist


class HistMerger:
    def __init__(self, req_entry: torch.Tensor, e_own: int, N: int, mode: str = "sparse",
                 group=None, accumulate=None):
        """req_entry: int32 [R] global entry ids of this rank's requests."""
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.group = group
        self.mode = mode
        self.N = N
        self.e_own = e_own
        self.e0, self.e1 = self.rank * e_own, (self.rank + 1) * e_own
        self.e_total = e_own * self.world
        dev = req_entry.device
        R = req_entry.numel()
        if accumulate is None:
            from . import sp
            accumulate = sp.accumulate_depths
        self.accumulate = accumulate
        r = torch.tensor([R], dtype=torch.int64, device=dev)
        dist.all_reduce(r, op=dist.ReduceOp.MAX, group=group)
        self.R, self.Rmax = R, int(r)
        # padded per-rank depth buffer: the LCP kernel writes [0, R); padding keeps entry -1
        self.lcp_pad = torch.full((max(self.Rmax, 1),), -1, dtype=torch.int32, device=dev)
        if mode == "sparse":
            ent_pad = torch.full((max(self.Rmax, 1),), -1, dtype=torch.int32, device=dev)
            ent_pad[:R] = req_entry
            self.g_ent = torch.empty(self.world * ent_pad.numel(), dtype=torch.int32, device=dev)
            dist.all_gather_into_tensor(self.g_ent, ent_pad, group=group)
            self.g_lcp = torch.empty_like(self.g_ent)
        elif mode == "allreduce":
            self.partial = torch.zeros(self.e_total, N + 1, dtype=torch.int32, device=dev)
        else:
            raise ValueError(mode)

    @property
    def lcp_out(self) -> torch.Tensor:
        """Buffer the LCP kernel writes this rank's depths into (first R slots)."""
        return self.lcp_pad

    def merge(self, hist_own: torch.Tensor, stream=None) -> torch.Tensor:
        """Add every rank's observations of the owned entries into hist_own [E_own][N+1].
        The collectives are issued with `stream` as the current stream, so they are ordered
        after the LCP kernel that filled lcp_out on that stream (NCCL runs on its own stream
        but waits on the current one)."""
        ctx = (torch.cuda.stream(stream) if stream is not None and hist_own.is_cuda
               else contextlib.nullcontext())
        with ctx:
            return self._merge(hist_own, stream)

    def _merge(self, hist_own: torch.Tensor, stream=None) -> torch.Tensor:
        if self.mode == "sparse":
            dist.all_gather_into_tensor(self.g_lcp, self.lcp_pad, group=self.group)
            self.accumulate(self.g_ent, self.g_lcp, self.e0, self.e1, self.N, hist_own,
                            stream=stream)
        else:
            dist.all_reduce(self.partial, group=self.group)
            hist_own.add_(self.partial[self.e0:self.e1])
            self.partial.zero_()
        return hist_own
