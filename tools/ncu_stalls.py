"""Per-instruction stall breakdown of an ncu report's source page (SASS view).

python tools/ncu_stalls.py REP.ncu-rep [--top N] [--range lo-hi]
Prints the stall-reason totals and the instructions with the most samples.
"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--range", default="")
args = ap.parse_args()
out = subprocess.run(["ncu", "-i", args.rep, "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = [r for r in rows[2:] if len(r) == len(hdr)]
if args.range:
    lo, hi = (int(x, 16) for x in args.range.split("-"))
    data = [r for r in data if lo <= int(r[ix["Address"]], 16) <= hi]
tot = {k: sum(float(r[ix[k]] or 0) for r in data) for k in reasons}
S = sum(tot.values()) or 1
print("stall totals:", ", ".join(f"{k[6:]} {100 * v / S:.1f}%" for k, v in
                                  sorted(tot.items(), key=lambda kv: -kv[1]) if v))
samp = lambda r: float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)  # noqa: E731
print(f"{'addr':>6} {'samples':>7}  top reasons  | source")
for r in sorted(data, key=samp, reverse=True)[: args.top]:
    rs = sorted(((float(r[ix[k]] or 0), k[6:]) for k in reasons), reverse=True)[:2]
    print(f"{r[ix['Address']]:>6} {samp(r):7.0f}  " + ", ".join(f"{k} {v:.0f}" for v, k in rs if v)
          + f"  | {r[ix['Source']].strip()[:70]}")
