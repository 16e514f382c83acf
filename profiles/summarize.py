"""Summarise an ncu report / launch list into profiles/*.json (run here, no GPU).

  python profiles/summarize.py gpurun_out/prof_full.ncu-rep profiles/r01_full.json
  python profiles/summarize.py --launches gpurun_out/launches.csv profiles/r01_launches.json
"""
import collections
import csv
import json
import subprocess
import sys

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "fma_pipe_active_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "xu_pipe_inst_pct": ("sm__inst_executed_pipe_xu.sum.pct_of_peak_sustained_active", 1),
    "alu_pipe_inst_pct": ("sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active", 1),
    "fma_pipe_inst_pct": ("sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active", 1),
    "warp_instructions": ("smsp__inst_executed.sum", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1),
    "smem_ld_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", 1),
    "smem_st_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", 1),
    "registers_per_thread": ("launch__registers_per_thread", 1),
    "grid_size": ("launch__grid_size", 1),
    "waves_per_sm": ("launch__waves_per_multiprocessor", 1),
    "sm_mhz": ("gpc__cycles_elapsed.avg.per_second", 1e-6),
}
STALLS = ["short_scoreboard", "long_scoreboard", "barrier", "wait", "math_pipe_throttle", "mio_throttle",
          "not_selected", "selected", "dispatch_stall", "no_instructions", "branch_resolving", "lg_throttle"]


def _num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        k = {"kernel": vals[h.index("Kernel Name")]}
        for name, (metric, scale) in KEYS.items():
            if metric in h:
                v = _num(vals[h.index(metric)])
                unit = units[h.index(metric)]
                if metric == "gpu__time_duration.sum" and unit in ("us", "usecond"):
                    scale = 1e-3
                if metric == "gpu__time_duration.sum" and unit in ("ms", "msecond"):
                    scale = 1.0
                if metric.startswith("dram__bytes") and unit in ("Kbyte", "KB"):
                    scale = 1e3
                if metric.startswith("dram__bytes") and unit in ("Mbyte", "MB"):
                    scale = 1e6
                if metric.startswith("dram__bytes") and unit in ("Gbyte", "GB"):
                    scale = 1e9
                if metric == "gpc__cycles_elapsed.avg.per_second" and unit in ("Ghz", "GHz"):
                    scale = 1e3
                k[name] = None if v is None else v * scale
        st = {}
        for s in STALLS:
            m = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if m in h:
                st[s] = _num(vals[h.index(m)])
        tot = sum(v for v in st.values() if v)
        k["stall_samples_pct"] = {s: round(100 * v / tot, 1) for s, v in st.items() if v} if tot else {}
        res.append(k)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


def launches(path, out, exclude=None):
    import re
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h, rows = rows[0], rows[1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows:
        if exclude and re.search(exclude, r[ki]):
            continue
        v = _num(r[vi])
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
        a = agg.setdefault(r[ki], [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    tot = sum(v[1] for v in agg.values())
    res = [{"kernel": k, "launches": c, "total_ms": round(t, 4), "share_pct": round(100 * t / tot, 2)}
           for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])]
    json.dump({"note": "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised): "
                       "compare shares, not absolute times" + (f"; excluded (not part of a step): {exclude}"
                                                                if exclude else ""),
               "kernels": res}, open(out, "w"), indent=1)
    for r in res:
        print(f"{r['launches']:5d} {r['total_ms']:9.3f} ms {r['share_pct']:6.2f}%  {r['kernel'][:90]}")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        full(sys.argv[1], sys.argv[2])
