"""Summarise ncu --set full reports into profiles/: a markdown table per report and ncu_traffic.json.

usage: python dbg/ncu_summary.py ROUND report1.ncu-rep [report2.ncu-rep ...]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
           "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active"]
SHORT = {"k_attn_fwd": "attn_fwd", "k_attn_bwd": "attn_bwd", "k_bwd_prep": "bwd_prep", "k_kv_image": "kv_image",
         "k_select_queries": "select_queries", "k_pool": "pool", "k_scores": "scores", "k_admit": "admit",
         "k_k2q": "k2q", "k_fill": "fill", "k_bwd_finalize": "bwd_finalize", "k_bwd_zero_pruned": "bwd_finalize",
         "k_partition_blocks": "partition", "k_partition_tokens": "partition"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
        "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                u = units[i]
                if isinstance(v, float) and u in UNIT:
                    v = v * UNIT[u]  # bytes -> bytes, time -> ms
                d[m] = v
        res.append(d)
    return res


def short(name):
    base = name.split("(")[0].split("<")[0].replace("void ", "").replace("bsa::", "").strip()
    return SHORT.get(base, base)


def main():
    rnd, reps = sys.argv[1], sys.argv[2:]
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    traffic_path = os.path.join(prof, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    tcfg = traffic.setdefault("wan1.3b_32k", {})
    for rep in reps:
        rows = rows_of(rep)
        name = os.path.splitext(os.path.basename(rep))[0]
        lines = [f"# ncu --set full summary: {name} (round {rnd})", "",
                 f"Source: `{os.path.basename(rep)}` (ncu --set full --clock-control none --import-source on, "
                 "bench.py wan1.3b_32k, one GPU). Durations are ncu replays (cold cache, serialised): compare "
                 "shares, not absolutes, with bench.py.", "",
                 "| kernel | grid | block | regs | ms | DRAM read MB | DRAM write MB | DRAM % | tensor pipe % | SM % | warps active % |",
                 "|---|---|---|---|---|---|---|---|---|---|---|"]
        for d in rows:
            g = lambda m, f="{:.1f}": (f.format(d[m]) if isinstance(d.get(m), float) else str(d.get(m, "-")))
            lines.append(f"| {short(d['kernel'])} | {g('launch__grid_size', '{:.0f}')} | {g('launch__block_size', '{:.0f}')} | "
                         f"{g('launch__registers_per_thread', '{:.0f}')} | {g('gpu__time_duration.sum', '{:.3f}')} | "
                         f"{d['dram__bytes_read.sum'] / 1e6:.1f} | {d['dram__bytes_write.sum'] / 1e6:.1f} | "
                         f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')} | "
                         f"{g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed')} | "
                         f"{g('sm__throughput.avg.pct_of_peak_sustained_elapsed')} | "
                         f"{g('sm__warps_active.avg.pct_of_peak_sustained_active')} |")
            tcfg[short(d["kernel"])] = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        open(os.path.join(prof, f"{rnd}_{name}.md"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
    json.dump(traffic, open(traffic_path, "w"), indent=1)


if __name__ == "__main__":
    main()
