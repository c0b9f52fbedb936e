"""Turn one `ncu --set full` report and one launch-list CSV (gpu__time_duration.sum per launch)
into the committed profile summaries:

  python tools/ncu_profiles.py --full gpurun_out/full.ncu-rep --launches gpurun_out/launches.csv \
      --tag r01b --cmd "python bench.py ..."

writes profiles/<tag>_ncu_full.txt (per-kernel metrics + top stall reasons),
profiles/<tag>_ncu_traffic.json (DRAM bytes per launch, read by bench.py) and
profiles/<tag>_launches.txt (launch counts, mean duration, share of the step)."""
import argparse
import collections
import csv
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__block_size", "launch__grid_size",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
# our kernels (ncu may print them without the sp:: namespace)
OURS = re.compile(r"\b(lcp_hist|accumulate_depths|row_stats|dp_hull|dp_hull_split|dp_lean|dp_place|"
                  r"eval_bcast|eval_p32|eval|gamma_observe|gamma_snapshot|grid_\w+|match|index_\w+)"
                  r"(_kernel)?\b")
UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "Tbyte": 1e12}


def short(name):
    n = name.split("(")[0].replace("void ", "").replace("sp::", "")
    return n.strip()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full")
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--cmd", default="")
    a = ap.parse_args()
    if a.full:
        raw = subprocess.run(["ncu", "-i", a.full, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout.splitlines()
        rows = list(csv.reader(raw))
        hdr, units = rows[0], rows[1]
        out_txt = [f"# ncu --set full --clock-control none: `{a.cmd}`",
                   f"# report: {os.path.basename(a.full)} (not committed); first captured launch per kernel", ""]
        traffic, pipes = {}, {}
        seen = set()
        for r in rows[2:]:
            kn = r[hdr.index("Kernel Name")]
            sk = short(kn)
            if sk in seen:
                continue
            seen.add(sk)
            out_txt.append(f"== {kn[:110]}")
            vals = {}
            for k in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    out_txt.append(f"   {k:76s} {r[i]} {units[i]}")
                    try:
                        vals[k] = float(r[i].replace(",", "")) * UNIT.get(units[i], 1.0)
                    except ValueError:
                        pass
            st = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                   float(r[i] or 0)) for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
            st.sort(key=lambda x: -x[1])
            out_txt.append("   top stall reasons (warps stalled per issued instruction):")
            for nme, v in st[:8]:
                out_txt.append(f"      {nme:30s} {v:.3f}")
            out_txt.append("")
            rd, wr = vals.get("dram__bytes_read.sum"), vals.get("dram__bytes_write.sum")
            traffic[sk] = {"dram_read_bytes": rd, "dram_write_bytes": wr,
                           "traffic_bytes": (rd + wr) if rd is not None and wr is not None else None,
                           "duration_ns": vals.get("gpu__time_duration.sum", 0) * 1e6
                           if "gpu__time_duration.sum" in vals else None,
                           "inst_executed": vals.get("smsp__inst_executed.sum")}
            pipes[sk] = {"issue_active_pct": vals.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                         "alu_pct": vals.get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                         "fma_pct": vals.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                         "lsu_pct": vals.get("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
                         "warps_active_pct": vals.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
                         "dram_throughput_pct": vals.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")}
        os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
        open(os.path.join(ROOT, "profiles", f"{a.tag}_ncu_full.txt"), "w").write("\n".join(out_txt) + "\n")
        json.dump(traffic, open(os.path.join(ROOT, "profiles", f"{a.tag}_ncu_traffic.json"), "w"), indent=1)
        json.dump(pipes, open(os.path.join(ROOT, "profiles", f"{a.tag}_ncu_pipes.json"), "w"), indent=1)
    if a.launches:
        lines = [ln for ln in open(a.launches) if not ln.startswith("==")]
        lr = list(csv.reader(lines))
        h = lr[0]
        iK, iV = h.index("Kernel Name"), h.index("Metric Value")
        agg = collections.OrderedDict()
        for x in lr[1:]:
            if "sp::" not in x[iK] and not OURS.search(x[iK]):
                continue
            k = short(x[iK])
            agg.setdefault(k, []).append(float(x[iV].replace(",", "")) / 1e6)   # ns -> ms
        tot = sum(sum(v) for v in agg.values())
        out = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, "
               f"serialised -- compare shares): `{a.cmd}`",
               f"{'kernel':44s} {'launches':>8s} {'mean ms':>10s} {'share':>8s}"]
        for k, v in agg.items():
            out.append(f"{k:44s} {len(v):8d} {sum(v) / len(v):10.3f} {sum(v) / tot * 100:7.1f}%")
        open(os.path.join(ROOT, "profiles", f"{a.tag}_launches.txt"), "w").write("\n".join(out) + "\n")
    if a.full:
        print(open(os.path.join(ROOT, "profiles", f"{a.tag}_ncu_full.txt")).read())


if __name__ == "__main__":
    main()
