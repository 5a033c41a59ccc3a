"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list into profiles/.

usage: python dbg/launch_summary.py ROUND launches.csv [timed_steps]
Only this library's kernels (namespace bsa::) are tabulated; the last `timed_steps` bench steps are used
(each step = one bsa_attn_fwd ... k_bwd_finalize sequence), shares are of the step's kernel time.
"""
import csv
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rnd, path = sys.argv[1], sys.argv[2]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "msecond": 1.0}
ours = []
for r in rows[1:]:
    name = r[ki]
    if "bsa::" not in name and not name.replace("void ", "").startswith("k_"):
        continue
    base = name.split("(")[0].replace("void ", "").replace("bsa::", "").split("<")[0].strip()
    ours.append((base, float(r[vi].replace(",", "")) * scale[r[ui]]))
# a step starts at the selection's first kernel (k_select_queries); keep the last `steps` of them
starts = [i for i, (b, _) in enumerate(ours) if b == "k_select_queries"]
first = starts[-steps] if len(starts) >= steps else 0
# the partition launch right before the step belongs to it
if first > 0 and ours[first - 1][0].startswith("k_partition"):
    first -= 1
if first > 1 and ours[first - 1][0].startswith("k_partition"):
    first -= 1
tail = ours[first:]
tot = sum(t for _, t in tail)
agg = {}
for b, t in tail:
    a = agg.setdefault(b, [0, 0.0])
    a[0] += 1
    a[1] += t
out = [f"# Launch list ({rnd}): bsa kernels of the last {steps} bench steps", "",
       f"Source: `{os.path.basename(path)}` = `ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_` over "
       "`python bench.py --steps 2 --warmup 3 --dense-steps 0 --e2e-steps 0 --no-cpu-baseline` (wan1.3b_32k). "
       "ncu serialises launches and runs them cold: compare shares with bench.py's live kernel_ms, not absolutes.",
       "", "| kernel | launches | ms per step | share of step |", "|---|---|---|---|"]
for b, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out.append(f"| {b} | {n // steps} | {t / steps:.3f} | {100 * t / tot:.1f}% |")
out.append(f"| **total** | {len(tail) // steps} | {tot / steps:.3f} | 100% |")
open(os.path.join(ROOT, "profiles", f"{rnd}_launches.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
