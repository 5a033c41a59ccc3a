"""Summarise an `ncu --page source --csv --print-source sass` export: stall totals and hottest SASS lines.
usage: python dbg/ncu_src.py file.csv [top]"""
import sys
import pandas as pd

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
df = pd.read_csv(path, skiprows=1)
num = lambda c: pd.to_numeric(df[c], errors="coerce").fillna(0)
stall_cols = [c for c in df.columns if c.startswith("stall_") and "Not Issued" not in c]
tot = {c: num(c).sum() for c in stall_cols}
S = sum(tot.values())
print("total samples", S)
for c, v in sorted(tot.items(), key=lambda x: -x[1])[:12]:
    print(f"  {c:28s} {v:9.0f} {100 * v / max(S, 1):5.1f}%")
df["samples"] = num("Warp Stall Sampling (All Samples)")
df["idx"] = range(len(df))
hot = df.sort_values("samples", ascending=False).head(top)
for _, r in hot.sort_values("idx").iterrows():
    stalls = sorted(((c[6:], num(c)[r.name]) for c in stall_cols), key=lambda x: -x[1])[:3]
    st = " ".join(f"{n}={v:.0f}" for n, v in stalls if v > 0)
    print(f"{r['idx']:5d} {r['Address']:>6} {r['samples']:7.0f}  {str(r['Source'])[:60]:60s} {st}")
