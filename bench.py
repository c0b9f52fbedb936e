#!/usr/bin/env python3
"""bench.py -- one step = one pass of the whole hot path over one batch.

Per rank and step (W5 by default = BASELINE.json configs[4], 16384 entries x N=32768 x M=64 per
GPU, weak scaling):
  a1+a2  sp_overlap_hist   over this rank's batch of new requests (20 per entry, end-spike law);
         the depths are merged into the resident per-entry histograms (1 GPU: accumulated in
         place; N GPUs: (entry, depth) pairs all-gathered over NCCL and scatter-added by the
         owner with sp_accumulate_depths, or --merge allreduce: dense int32 NCCL all-reduce)
  a3-a5  sp_place_checkpoints on the owned histograms (dense depth-mode laws, n ~ U[8192,16384]
         draws per entry plus the new requests), cost_by_budget for the V_0..V_M frontier
  a6     sp_expected_recompute for the balanced (M) and block (B = 64, 128) baselines
Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DP cells/s (entries*N*M)"
TRAFFIC_JSON = "r02i_ncu_traffic.json"   # ncu capture of the current kernels (tools/ncu_profiles.py)
PIPES_JSON = "r02i_ncu_pipes.json"       # the same capture: issue / ALU / FMA / LSU pipe %


def dp_update_cost():
    """Minimal amortised SASS of one hull update on the INT pipes, and the
    SM-cycles it needs at the lane rates measured on this pool's B200 by tools/int_rate.cu
    (profiles/r02_int_rate.json).  Per update, with b = 1.905 back tests and f = 1.091 front
    tests (W5 rows, tools/hull_stats.c): intercept 1 IMAD; per back test 2 IADD deltas, 2
    IMAD.WIDE, 1 ISETP; per back pop (b - 1) and front pop (f - 1) one ring LDS + 1 address
    op; push 2 STS + 1 address op; per front test 1 IMAD + 1 ISETP; query 1 IMAD; counters 1."""
    b, f = 1.905, 1.091
    alu = 2 * b + b + (b - 1) + (f - 1) + 1 + f + 1
    imad = 1 + f + 1
    imad_wide = 2 * b
    lsu = (b - 1) + 2 + (f - 1)
    rates = {"alu": 63.6, "fma_imad": 63.5, "imad_wide": 26.8, "lsu": 31.1, "issue": 128.0}
    t = {"alu": alu / rates["alu"],
         "fma": imad / rates["fma_imad"] + imad_wide / rates["imad_wide"],
         "lsu": lsu / rates["lsu"],
         "issue": (alu + imad + imad_wide + lsu) / rates["issue"]}
    binding = max(t, key=t.get)
    return {"ops": {"alu": round(alu, 3), "imad": round(imad, 3), "imad_wide": round(imad_wide, 3),
                    "lsu": round(lsu, 3)},
            "rates": rates, "clk_per_update_per_sm": t[binding], "binding": binding}
UNIT = "cells/s"


def _kget(d, prefix):
    """The entry of a per-kernel ncu summary for the int32 hull kernel, whatever the spelling of
    its trailing template arguments (", 0>" / ", false>" / ">")."""
    for k in (prefix + ">", prefix + ", 0>", prefix + ", false>"):
        if k in d:
            return d[k]
    return {}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="W5", choices=["W2", "W3", "W4", "W5"])
    ap.add_argument("--entries", type=int, default=None,
                    help="entries in total (strong) or per GPU (weak); default: the config's")
    ap.add_argument("--merge", default="sparse", choices=["sparse", "allreduce"])
    ap.add_argument("--dp-hist", default="dense", choices=["dense", "ones", "accum"],
                    help="DP input rows: dense depth-mode (default, SURVEY 8(d) W5); ones: all-ones "
                         "rows (full support, the D&C worst case and Thm 1's uniform law); accum: "
                         "accumulated rows with n ~ U[1.2e5, 1.8e5] draws (past the int32 guard)")
    ap.add_argument("--weights", default="i32", choices=["i32", "f64"],
                    help="i32: integer counts (exact int32 path, the default); f64: the paper's "
                         "probability weights (a7) kept by the gamma-estimator (f2, P:323-343, "
                         "P:380): each step's LCPs are observed into fp64 rows W (initialised from "
                         "the dense rows) and the fp64 DP and evaluation run on W (N = 1 only)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's entries split over the GPUs (BASELINE configs[4]); "
                         "weak: the config's entries on every GPU")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=8, help="entry blocks of the pipelined e2e")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle wall time")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ---------------------------------------------------------------------------------------------
# clocks (B200_PROFILING.md "clocks DURING the timed region")
# ---------------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def wait(self, event):
        event.synchronize()

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in out.strip().splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "samples": len(sm),
                "reasons": sorted(reasons)}


class NvmlClockSampler:
    """Samples NVML from the host thread itself while it waits for the timed region's end event
    (query + sample every ~3 ms), so even a ~200 ms region gets tens of samples taken while the
    kernels run; ClockSampler (nvidia-smi) is the fallback."""
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu: int):
        import pynvml
        import torch
        self.nv = pynvml
        pynvml.nvmlInit()
        try:
            pr = torch.cuda.get_device_properties(gpu)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu)
        self.bits = dict(zip(self.NAMES, (pynvml.nvmlClocksEventReasonHwSlowdown,
                                          pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                                          pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                                          pynvml.nvmlClocksEventReasonSwPowerCap)))
        self.sm, self.reasons = [], set()

    def _sample(self):
        nv = self.nv
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        for nm, b in self.bits.items():
            if r & b:
                self.reasons.add(nm)

    def start(self):
        pass

    def wait(self, event):
        """Sample until `event` (recorded at the end of the timed region) has completed."""
        while True:
            self._sample()
            if event.query():
                break
            time.sleep(0.003)

    def stop(self):
        smax = float(self.nv.nvmlDeviceGetMaxClockInfo(self.h, self.nv.NVML_CLOCK_SM))
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": smax,
                "samples": len(self.sm), "reasons": sorted(self.reasons), "source": "nvml"}


def clock_sampler(gpu: int):
    try:
        return NvmlClockSampler(gpu)
    except Exception:
        return ClockSampler(gpu)


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ---------------------------------------------------------------------------------------------
# the CPU oracle as baseline (cpu_baseline leg and --impl reference)
# ---------------------------------------------------------------------------------------------
def oracle_sample_step(oracle, sample, nthreads):
    """One oracle pass over a bounded sample: LCP loop + CHT DP + baseline evaluation."""
    t0 = time.perf_counter()
    hist = sample["hist"].copy()
    oracle.lcp_hist(sample["entry_tokens"], sample["entry_off"], sample["req_tokens"],
                    sample["req_off"], sample["req_entry"], sample["N"], n_entries=hist.shape[0],
                    hist=hist, nthreads=nthreads)
    t1 = time.perf_counter()
    oracle.place_batch(hist, sample["M"], "cht", nthreads=nthreads)
    t2 = time.perf_counter()
    oracle.eval_batch(hist, sample["bpos"], sample["bnpos"], broadcast=True, nthreads=nthreads)
    t3 = time.perf_counter()
    return t3 - t0, (t1 - t0, t2 - t1, t3 - t2)


def build_oracle_sample(args, n_entries):
    """Host copy of a bounded sample of the workload (the generator's inputs, never CUDA
    outputs): the first n_entries entries with their requests and dense histograms."""
    import numpy as np
    import torch
    from paper_2605_05219_b200 import sp
    from paper_2605_05219_b200 import workload as wl
    cfg = wl.CONFIGS[args.workload]
    scfg = wl.scaled(cfg, n_entries)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    tr = wl.make_trace(scfg, seed=args.seed, device=dev)
    if cfg.dense_n:
        hist = wl.make_dense_hist(scfg, seed=args.seed, device=dev)
    else:
        hist = torch.zeros(n_entries, cfg.N + 1, dtype=torch.int32, device=dev)
    budgets = cfg.M_sweep if cfg.M_sweep else (cfg.M,)
    sets = [sp_balanced(cfg.N, m) for m in budgets] + [sp_block(cfg.N, B) for B in (64, 128)]
    width = max(len(s) for s in sets)
    bpos = np.zeros((len(sets), width), np.int32)
    for i, s in enumerate(sets):
        bpos[i, :len(s)] = s
    return dict(entry_tokens=tr["entry_tokens"].cpu().numpy(),
                entry_off=tr["entry_off"].cpu().numpy(), req_tokens=tr["req_tokens"].cpu().numpy(),
                req_off=tr["req_off"].cpu().numpy(), req_entry=tr["req_entry"].cpu().numpy(),
                hist=hist.cpu().numpy(), N=cfg.N, M=cfg.M, bpos=bpos,
                bnpos=np.array([len(s) for s in sets], np.int32), E=n_entries)


def sp_balanced(N, M):
    # Table 1 balanced schedule, generated on the host for the oracle sample
    return [(i * (N + 1)) // (M + 1) for i in range(1, M + 1)]


def sp_block(N, B):
    return [B * i for i in range(1, N // B + 1)]


def calibrate_sample(args, oracle, nthreads, target_s):
    """Pick a sample size whose oracle step takes ~target_s seconds of wall time."""
    cfg_E = (args.entries or __import__("paper_2605_05219_b200.workload",
                                        fromlist=["CONFIGS"]).CONFIGS[args.workload].n_entries)
    n = min(2 * nthreads, cfg_E)
    s = build_oracle_sample(args, n)
    dt, _ = oracle_sample_step(oracle, s, nthreads)
    n2 = int(min(cfg_E, max(n, n * target_s / max(dt, 1e-3))))
    n2 = max(nthreads, (n2 // nthreads) * nthreads) if n2 >= nthreads else n2
    if n2 != n:
        s = build_oracle_sample(args, n2)
    return s


def cpu_baseline(args, nthreads):
    import oracle
    oracle.build()
    s = calibrate_sample(args, oracle, nthreads, args.cpu_seconds)
    dt, parts = oracle_sample_step(oracle, s, nthreads)
    cells = s["E"] * s["N"] * s["M"]
    return {"value": cells / dt, "unit": UNIT, "cores": nthreads, "kind": "oracle",
            "sample": (f"first {s['E']} entries of {args.workload} (full N={s['N']}, M={s['M']}, "
                       f"their {len(s['req_off']) - 1} requests): literal LCP loop + paper's "
                       f"CHT DP (int64/__int128) + definitional baseline evaluation, "
                       f"{nthreads} pthreads"),
            "seconds": dt, "seconds_lcp_dp_eval": parts,
            "dp_only_cells_per_s": cells / parts[1] if parts[1] > 0 else None,
            "cpu_model": cpu_model()}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    """--impl reference: the oracle (the tier's reference arm) on the host cores."""
    world, rank, _ = env_rank()
    if rank != 0:
        return
    import oracle
    oracle.build()
    nthreads = os.cpu_count() or 1
    per_step = max(2.0, min(20.0, 150.0 / max(args.steps + args.warmup, 1)))
    s = calibrate_sample(args, oracle, nthreads, per_step)
    for _ in range(args.warmup):
        oracle_sample_step(oracle, s, nthreads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_sample_step(oracle, s, nthreads)
    dt = time.perf_counter() - t0
    cells = s["E"] * s["N"] * s["M"] * args.steps
    v = cells / dt
    cfg = workload_config(args, max(args.gpus, world), None)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": nthreads, "kind": "oracle",
                             "sample": f"first {s['E']} entries of {args.workload} per step",
                             "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(args, world, extra):
    from paper_2605_05219_b200 import workload as wl
    cfg = wl.CONFIGS[args.workload]
    E_tot, E = plan_entries(args, cfg, world)
    d = {"workload": f"{args.workload}: {E_tot} entries x N={cfg.N} x M={cfg.M}"
                     + (f" ({E}/GPU)" if world > 1 else ""),
         "entries_per_gpu": E, "entries_total": E_tot, "N": cfg.N, "M": cfg.M,
         "requests_per_entry": cfg.req_per_entry, "lcp_law": cfg.shape,
         "dp_hist": ({"ones": "all-ones rows (full support) + the step's requests",
                      "accum": f"accumulated depth-mode rows, n~U[120000, 180000] draws/entry, "
                               f"{cfg.dense_shape} laws, + the step's requests"}.get(
                         getattr(args, "dp_hist", "dense"))
                     or (f"dense depth-mode, n~U{list(cfg.dense_n)} draws/entry, {cfg.dense_shape} "
                         f"laws, + the step's requests" if cfg.dense_n else "from the LCP requests")),
         "weights": ("f64: gamma-estimator rows W (gamma = 0.99), initialised from the dense "
                     "rows, the step's LCPs observed into them (P:323-343, P:380)"
                     if getattr(args, "weights", "i32") == "f64" else "int32 counts"),
         "parallelism": f"entries sharded over {world} GPU(s) ({args.scaling} scaling)",
         "merge": None if world == 1 else args.merge,
         "l2": "inputs larger than L2 (request tokens and histograms >> 126 MB)"}
    if extra:
        d.update(extra)
    return d


# ---------------------------------------------------------------------------------------------
# one rank's resident state and step (shared by the GPU arm and the gloo CPU test of the N > 1
# path, tests/test_bench_gloo.py, which passes CPU stand-ins as `ops`)
# ---------------------------------------------------------------------------------------------
def plan_entries(args, cfg, world):
    """(E_total, E_own).  Strong scaling (default): BASELINE.json configs[4] is "16k entries ...
    sharded across 8xB200", so the total is the config's and each rank owns E_total / N.
    Weak: each rank owns the config's entry count."""
    if args.scaling == "strong":
        E_tot = args.entries or cfg.n_entries
        if E_tot % world:
            raise SystemExit(f"strong scaling: {E_tot} entries do not split over {world} ranks")
        return E_tot, E_tot // world
    E_own = args.entries or cfg.n_entries
    return E_own * world, E_own


class HotPath:
    """Rank `rank` of `world`: owns entries [rank E_own, (rank+1) E_own) of E_tot, holds their
    resident histograms, this rank's batch of new requests (routed at random),
    the outputs and the DP workspace.  step(): a1+a2 LCP-histogram of the batch, the merge
    (world > 1: the one exchange step, paper_2605_05219_b200.dist), a3-a5 DP on the owned
    entries, a6 baseline evaluation."""

    def __init__(self, cfg, E_tot, E_own, world, rank, merge, seed, dev, ops=None,
                 dp_hist="dense", weights="i32"):
        import torch
        from paper_2605_05219_b200 import workload as wl
        if ops is None:
            from paper_2605_05219_b200 import sp as ops
        self.ops, self.world, self.merge_mode = ops, world, merge
        self.E_tot, self.E_own, self.N, self.M = E_tot, E_own, cfg.N, cfg.M
        self.e0 = rank * E_own
        N, M = cfg.N, cfg.M
        tcfg = wl.scaled(cfg, E_tot)
        self.tr = tr = wl.make_trace(tcfg, seed=seed, device=dev, world=world, rank=rank)
        self.R = tr["req_off"].numel() - 1
        if dp_hist == "ones":
            self.hist = wl.uniform_hist(E_own, N, device=dev)
        elif dp_hist == "accum":
            import dataclasses
            acfg = dataclasses.replace(tcfg, dense_n=(120000, 180000))
            self.hist = wl.make_dense_hist(acfg, seed=seed, device=dev, entry_begin=self.e0,
                                           n_entries=E_own)
        elif cfg.dense_n:
            self.hist = wl.make_dense_hist(tcfg, seed=seed, device=dev, entry_begin=self.e0,
                                           n_entries=E_own)
        else:
            self.hist = torch.zeros(E_own, N + 1, dtype=torch.int32, device=dev)
        self.gest = None
        if weights == "f64":
            # a7 on the paper's probability weights: the gamma-estimator's rows W (f2; its
            # observe kernel folds each step's LCPs in, misses skipped, R15), W initialised
            # from the resident counts; the DP and the evaluation run on W (scale invariant)
            assert world == 1, "--weights f64 runs at N = 1"
            self.gest = ops.GammaEstimator(E_own, N, gamma=0.99, device=dev)
            self.gest.W.copy_(self.hist)
            re_ = tr["req_entry"].long()
            bounds = torch.arange(E_own + 1, device=dev, dtype=torch.int64)
            self.obs_off = torch.searchsorted(re_, bounds).to(torch.int64)
        cdt = torch.float64 if weights == "f64" else torch.int64
        budgets = cfg.M_sweep if cfg.M_sweep else (M,)
        self.bpos, self.bnpos, self.labels = ops.baseline_sets(N, budgets=budgets,
                                                               blocks=(64, 128), device=dev)
        self.S = S = self.bpos.shape[0]
        self.positions = torch.empty(E_own, M, dtype=torch.int32, device=dev)
        self.npos = torch.empty(E_own, dtype=torch.int32, device=dev)
        self.cost = torch.empty(E_own, dtype=cdt, device=dev)
        self.cbb = torch.empty(E_own, M + 1, dtype=cdt, device=dev)
        self.bcost = torch.empty(E_own, S, dtype=cdt, device=dev)
        self.bworst = torch.empty(E_own, S, dtype=torch.int32, device=dev)
        self.ws = torch.empty(ops.place_checkpoints_workspace_bytes(E_own, N, M),
                              dtype=torch.uint8, device=dev)
        self.lcp = torch.full((max(self.R, 1),), -1, dtype=torch.int32, device=dev)
        self.merger = None
        if world > 1:
            from paper_2605_05219_b200.dist import HistMerger
            self.merger = HistMerger(tr["req_entry"], E_own, N, mode=merge,
                                     accumulate=ops.accumulate_depths)

    def step(self, stream=None, marks=None):
        ops, tr, N, M = self.ops, self.tr, self.N, self.M
        if marks:
            marks[0].record(stream)
        # a1 + a2
        if self.gest is not None:   # f64: the LCPs only; the estimator takes them below
            ops.overlap_hist(tr["entry_tokens"], tr["entry_off"], tr["req_tokens"], tr["req_off"],
                             tr["req_entry"], N, lcp_out=self.lcp, n_entries=self.E_tot,
                             stream=stream, with_hist=False)
        elif self.world == 1:
            ops.overlap_hist(tr["entry_tokens"], tr["entry_off"], tr["req_tokens"], tr["req_off"],
                             tr["req_entry"], N, hist=self.hist, lcp_out=self.lcp,
                             n_entries=self.E_tot, stream=stream)
        elif self.merge_mode == "sparse":
            ops.overlap_hist(tr["entry_tokens"], tr["entry_off"], tr["req_tokens"], tr["req_off"],
                             tr["req_entry"], N, lcp_out=self.merger.lcp_out,
                             n_entries=self.E_tot, stream=stream, with_hist=False)
        else:
            ops.overlap_hist(tr["entry_tokens"], tr["entry_off"], tr["req_tokens"], tr["req_off"],
                             tr["req_entry"], N, hist=self.merger.partial, lcp_out=self.lcp,
                             n_entries=self.E_tot, stream=stream)
        if marks:
            marks[1].record(stream)
        # merge (the one exchange step)
        if self.world > 1:
            self.merger.merge(self.hist, stream=stream)
        if self.gest is not None:   # f2: observe the step's depths into W
            self.gest.observe(self.obs_off, self.lcp, stream=stream)
        if marks:
            marks[2].record(stream)
        w = self.hist if self.gest is None else self.gest.W
        # a3 - a5
        ops.place_checkpoints(w, M, positions=self.positions, n_positions=self.npos,
                              cost=self.cost, cost_by_budget=self.cbb, workspace=self.ws,
                              stream=stream)
        if marks:
            marks[3].record(stream)
        # a6
        ops.expected_recompute(w, self.bpos, self.bnpos, broadcast=True, cost=self.bcost,
                               worst=self.bworst, stream=stream)
        if marks:
            marks[4].record(stream)


# ---------------------------------------------------------------------------------------------
# the GPU arm
# ---------------------------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2605_05219_b200 import build as bld
    from paper_2605_05219_b200 import sp
    from paper_2605_05219_b200 import workload as wl

    world, rank, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        bld.build()
    if world > 1:
        dist.barrier()
    sp.lib()

    cfg = wl.CONFIGS[args.workload]
    E_tot, E_own = plan_entries(args, cfg, world)
    e0 = rank * E_own
    N, M = cfg.N, cfg.M
    hp = HotPath(cfg, E_tot, E_own, world, rank, args.merge, args.seed, dev,
                 dp_hist=args.dp_hist, weights=args.weights)
    tr, hist, R = hp.tr, hp.hist, hp.R
    positions, npos, cost, cbb, bcost, bworst = (hp.positions, hp.npos, hp.cost, hp.cbb,
                                                 hp.bcost, hp.bworst)
    bpos, bnpos, S, ws, lcp = hp.bpos, hp.bnpos, hp.S, hp.ws, hp.lcp

    # tokens examined by the LCP (generator depths): sum min(t+1, len, L_e)
    d = torch.minimum(tr["depth"].to(torch.int64), torch.tensor(N, device=dev))
    rlen = tr["req_off"][1:] - tr["req_off"][:-1]
    Le = tr["L"][tr["req_entry"].long()]
    lim = torch.minimum(torch.minimum(rlen, Le), torch.tensor(N, device=dev))
    examined = torch.minimum(d + 1, lim)
    tokens_examined = int(examined.sum())
    # algorithmic HBM bytes of the LCP kernel: request + entry tokens examined (entry tokens
    # once per entry: max over its requests), offsets/ids, one histogram update per request
    ent_max = torch.zeros(E_tot, dtype=torch.int64, device=dev)
    ent_max.scatter_reduce_(0, tr["req_entry"].long(), examined, reduce="amax")
    lcp_bytes = 4 * tokens_examined + 4 * int(ent_max.sum()) + R * (4 + 16 + 16 + 4 + 4)

    stream = torch.cuda.current_stream(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    req_tokens, req_off, req_entry = tr["req_tokens"], tr["req_off"], tr["req_entry"]

    def step(marks=None):
        hp.step(stream=stream, marks=marks)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- warm-up ---------------------------------------------------------------------------
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stats = sp.dp_stats(ws)
    assert (npos >= 0).all(), "DP flagged an entry (negative n_positions)"

    # ---- timed region (device-resident inputs) -----------------------------------------------
    marks = [[ev() for _ in range(5)] for _ in range(args.steps)]
    clocks = clock_sampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    t_start, t_end = ev(), ev()
    t_start.record(stream)
    for k in range(args.steps):
        step(marks[k])
    t_end.record(stream)
    clocks.wait(t_end)          # samples clocks while the timed steps run
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = t_start.elapsed_time(t_end)
    stage = np.array([[marks[k][i].elapsed_time(marks[k][i + 1]) for i in range(4)]
                      for k in range(args.steps)])          # lcp, merge, dp, eval (ms)
    t = torch.tensor([ms] + list(stage.sum(0)), dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, lcp_ms, merge_ms, dp_ms, eval_ms = [float(x) for x in t.cpu()]

    # ---- e2e: through the C ABI with the step's inputs in pinned HOST memory -----------------
    e2e = None
    if not args.no_e2e:
        h_tok = torch.empty(req_tokens.shape, dtype=torch.int32, pin_memory=True)
        h_tok.copy_(req_tokens)
        h_off = req_off.cpu().pin_memory()
        h_ent = req_entry.cpu().pin_memory()
        o_pos = torch.empty(positions.shape, dtype=torch.int32, pin_memory=True)
        o_npos = torch.empty(npos.shape, dtype=torch.int32, pin_memory=True)
        o_cost = torch.empty(cost.shape, dtype=cost.dtype, pin_memory=True)
        o_bcost = torch.empty(bcost.shape, dtype=bcost.dtype, pin_memory=True)
        o_cbb = torch.empty(cbb.shape, dtype=cbb.dtype, pin_memory=True)
        bi = (h_tok.numel() * 4 + h_off.numel() * 8 + h_ent.numel() * 4)
        bo = (o_pos.numel() * 4 + o_npos.numel() * 4 + o_cost.numel() * 8 + o_bcost.numel() * 8
              + o_cbb.numel() * 8)

        def e2e_step():
            req_tokens.copy_(h_tok, non_blocking=True)
            req_off.copy_(h_off, non_blocking=True)
            req_entry.copy_(h_ent, non_blocking=True)
            step()
            o_pos.copy_(positions, non_blocking=True)
            o_npos.copy_(npos, non_blocking=True)
            o_cost.copy_(cost, non_blocking=True)
            o_bcost.copy_(bcost, non_blocking=True)
            o_cbb.copy_(cbb, non_blocking=True)

        run_e2e = e2e_step
        if world == 1 and args.e2e_chunks > 1:
            # pipelined through the same ABI calls: the request tokens of entry block c+1 cross
            # PCIe (copy stream) while blocks <= c run LCP -> DP -> evaluation (compute stream);
            # requests are grouped by entry, so a block's requests and tokens are contiguous
            C = args.e2e_chunks
            h_ent_np = h_ent.numpy()
            eb = [E_own * c // C for c in range(C + 1)]
            rb = [int(np.searchsorted(h_ent_np, x, side="left")) for x in eb]
            tb = [int(h_off[r]) for r in rb]
            cstream = torch.cuda.Stream(dev)
            cev = [ev() for _ in range(C)]

            def e2e_pipelined():
                req_off.copy_(h_off, non_blocking=True)
                req_entry.copy_(h_ent, non_blocking=True)
                cstream.wait_stream(stream)
                with torch.cuda.stream(cstream):
                    for c in range(C):
                        req_tokens[tb[c]:tb[c + 1]].copy_(h_tok[tb[c]:tb[c + 1]], non_blocking=True)
                        cev[c].record(cstream)
                for c in range(C):
                    stream.wait_event(cev[c])
                    r0, r1, a0, a1 = rb[c], rb[c + 1], eb[c], eb[c + 1]
                    g = hp.gest
                    if r1 > r0:
                        sp.overlap_hist(tr["entry_tokens"], tr["entry_off"], req_tokens,
                                        req_off[r0:r1 + 1], req_entry[r0:r1], N,
                                        hist=hist if g is None else None,
                                        lcp_out=lcp[r0:r1], n_entries=E_tot, stream=stream,
                                        with_hist=g is None)
                    w = hist
                    if g is not None:   # f64: observe the block's depths, then solve on W
                        sp.gamma_observe(g.W[a0:a1], g.t[a0:a1], g.tau[a0:a1],
                                         hp.obs_off[a0:a1 + 1], lcp, g.gamma, stream)
                        w = g.W
                    sp.place_checkpoints(w[a0:a1], M, positions=positions[a0:a1],
                                         n_positions=npos[a0:a1], cost=cost[a0:a1],
                                         cost_by_budget=cbb[a0:a1], workspace=ws, stream=stream)
                    sp.expected_recompute(w[a0:a1], bpos, bnpos, broadcast=True,
                                          cost=bcost[a0:a1], worst=bworst[a0:a1], stream=stream)
                    o_pos[a0:a1].copy_(positions[a0:a1], non_blocking=True)
                    o_npos[a0:a1].copy_(npos[a0:a1], non_blocking=True)
                    o_cost[a0:a1].copy_(cost[a0:a1], non_blocking=True)
                    o_bcost[a0:a1].copy_(bcost[a0:a1], non_blocking=True)
                    o_cbb[a0:a1].copy_(cbb[a0:a1], non_blocking=True)

            run_e2e = e2e_pipelined
        run_e2e()
        torch.cuda.synchronize()
        barrier()
        a, b = ev(), ev()
        a.record(stream)
        for _ in range(args.steps):
            run_e2e()
        b.record(stream)
        torch.cuda.synchronize()
        barrier()
        e_ms = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e_ms = float(e_ms)
        e2e = {"value": E_tot * N * M * args.steps / (e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": bi * world, "d2h_bytes_per_step": bo * world,
               "ms_per_step": e_ms / args.steps,
               "pipeline": (f"{args.e2e_chunks} entry blocks, H2D on a copy stream overlapped "
                            f"with LCP/DP/eval" if world == 1 and args.e2e_chunks > 1
                            else "serial")}

    # ---- numbers -------------------------------------------------------------------------
    tok_all = torch.tensor([tokens_examined, lcp_bytes], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tok_all)
    tokens_all, lcp_bytes_all = [float(x) for x in tok_all.cpu()]
    K = args.steps
    value = E_tot * N * M * K / (ms_max / 1e3)
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    wbytes = 8 if args.weights == "f64" else 4
    eval_bytes = E_own * (N + 1) * wbytes + E_own * S * (8 + 4)   # rows read once; costs + worst
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    # DP roofline: INT-pipe bound, no tensor cores (min-plus).  The algorithmic
    # unit is one hull update -- one (layer, support row) step of the paper's monotone CHT
    # -- counted exactly by the kernel (support rows x M).  Peak = the minimal
    # amortised SASS of an update (dp_update_cost) on the INT pipes at the rates measured by
    # tools/int_rate.cu on this B200 (profiles/r02_int_rate.json).
    upd = dp_update_cost()
    updates = stats["hull_event_rows"] * M
    traffic, pipes = {}, {}
    f64 = args.weights == "f64"
    try:   # DRAM bytes and pipe utilisation per launch from the committed `ncu --set full`
        if args.workload == "W5" and E_own == 16384 and args.dp_hist == "dense" and not f64:
            traffic = json.load(open(os.path.join(ROOT, "profiles", TRAFFIC_JSON)))
            pipes = json.load(open(os.path.join(ROOT, "profiles", PIPES_JSON)))
    except Exception:
        traffic, pipes = traffic or {}, {}
    dp_launch_s = dp_ms / K / 1e3
    achieved = updates / dp_launch_s / 1e9
    peak = sms * sm_max * 1e6 / upd["clk_per_update_per_sm"] / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_max / K, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": ("f64 (double-double P_j and costs, reading R10)" if f64
                                                  else "int32-exact (int64 costs)"),
        "data": "synthetic (seeded; SURVEY 8(d) recipe)",
        "config": workload_config(args, world, None),
        "lcp_tokens_per_s": tokens_all * K / (lcp_ms / 1e3),
        "stage_ms_per_step": {"lcp_hist": lcp_ms / K,
                              ("gamma_observe" if f64 else "merge"): merge_ms / K,
                              "dp": dp_ms / K, "eval": eval_ms / K},
        "roofline": {"bound": "alu", "kernel": ("dp_hull_kernel<double, 2, double>" if f64 else
                                                         "dp_hull_kernel<int32> (dp_hull_split_kernel for < 1.5 entries per resident warp)"), "achieved": achieved,
                     "peak": peak, "unit": "Gupd/s", "frac": achieved / peak,
                     "traffic": _kget(traffic, "dp_hull_kernel<int, 2, int").get("traffic_bytes"),
                     "work": f"{updates} hull updates per launch = {stats['hull_event_rows']} "
                             f"support rows x M (support rows = {stats['hull_event_rows'] / max(1, stats['entries_hull']) / N:.3f} "
                             f"of N per entry; zero-count rows are exact no-ops); "
                             f"{stats['entries_hull']} entries on the hull kernel "
                             f"({stats.get('entries_hull_big', 0)} in its large-hull mode), "
                             f"{E_own - stats['entries_hull']} on the D&C fallback "
                             f"({stats['evaluations']} candidate evaluations)",
                     "peak_basis": (f"{sms} SMs x {sm_max:.0f} MHz / {upd['clk_per_update_per_sm']:.4f} "
                                    f"SM-cycles per update (binding pipe: {upd['binding']}); "
                                    f"minimal amortised update = {upd['ops']} at measured lanes/clk/SM "
                                    f"{upd['rates']}"
                                    + ("; the int32 step's peak: the fp64 step's own minimal SASS "
                                       "(DFMA / DSETP) is not derived" if f64 else "")),
                     "pipes_ncu": _kget(pipes, "dp_hull_kernel<int, 2, int") or None,
                     "support_fraction": stats["hull_event_rows"] / max(1, stats["entries_hull"]) / N
                     if stats["entries_hull"] else None,
                     "support_updates_per_s": updates / dp_launch_s,
                     "dense_cells_per_s": E_own * N * M / dp_launch_s},
        "roofline_lcp": {"bound": "hbm", "kernel": "lcp_hist_kernel",
                         "achieved": lcp_bytes_all * K / (lcp_ms / 1e3) / 1e9 / world,
                         "peak": hbm_peak, "unit": "GB/s",
                         "frac": lcp_bytes_all * K / (lcp_ms / 1e3) / 1e9 / world / hbm_peak,
                         "traffic": traffic.get("lcp_hist_kernel", {}).get("traffic_bytes"),
                         "algorithmic_bytes": lcp_bytes_all / world},
        # a6: reads every histogram row once, writes E x S costs (eval_bcast_kernel for <= 4
        # broadcast sets whose l tables fit shared memory, else eval_p32_kernel)
        "roofline_eval": {"bound": "hbm", "kernel": (f"eval_bcast_f64_kernel<{S}>" if f64 else
                                                     f"eval_bcast_kernel<{S}>"
                                                     if S <= 4 and S * (N + 1 + 384) * 2 <= 200 * 1024
                                                     else "eval_p32_kernel<uint16_t, 256>"),
                          "achieved": eval_bytes * K / (eval_ms / 1e3) / 1e9,
                          "peak": hbm_peak, "unit": "GB/s",
                          "frac": eval_bytes * K / (eval_ms / 1e3) / 1e9 / hbm_peak,
                          "traffic": traffic.get(f"eval_bcast_kernel<{S}>", {}).get("traffic_bytes"),
                          "algorithmic_bytes": eval_bytes},
        "dp_paths": {k: v for k, v in stats.items()},
        # per step: lcp_hist, row_stats (+ CUB's radix-sort kernels), dp_hull<int32> (or
        # dp_hull_split for small batches), its large-hull mode and dp_hull<int64> (their lists;
        # each exits at once when empty), dp_place (the D&C list; ditto), eval (+
        # accumulate_depths for the sparse merge).  f64: lcp_hist, gamma_observe, row_stats,
        # dp_hull<double>, dp_place, eval.  Counted: our kernels only.
        "gpu_launches": K * (6 if f64 else
                             7 + (1 if world > 1 and args.merge == "sparse" else 0)),
        "clocks": clk,
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:   # (N = 1 only)
        line["cpu_baseline"] = cpu_baseline(args, os.cpu_count() or 1)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
