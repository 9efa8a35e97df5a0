"""Summarise an ncu source page (SASS): top instructions by executed count and by stall samples.
usage: python tools/sass_hot.py report.ncu-rep [kernel-regex] [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 2 and sys.argv[2]:
    args += ["-k", "regex:" + sys.argv[2]]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
hi = rows.index(hdr)
body = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
ix = {k: i for i, k in enumerate(hdr)}
def num(r, k):
    try: return float(r[ix[k]])
    except: return 0.0
tot_i = sum(num(r, "Instructions Executed") for r in body)
tot_s = sum(num(r, "Warp Stall Sampling (All Samples)") for r in body)
print(f"{len(body)} SASS lines, {tot_i:.0f} warp instructions, {tot_s:.0f} samples")
for i, r in enumerate(body):
    r.append(i)
print("-- by stall samples")
for r in sorted(body, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:top]:
    print(f"{r[-1]:5d} {num(r,'Warp Stall Sampling (All Samples)'):7.0f} {num(r,'Instructions Executed'):9.0f}  {r[1].strip()[:70]}")
