"""Stall-reason breakdown of an ncu report's SASS page (needs --import-source / --set full).

    python tools/ncu_stalls.py rep.ncu-rep [--top N] [--window ADDR_LO ADDR_HI]

Prints the kernel-wide stall totals by reason and the top-N instructions by samples with
their dominant reasons.
"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--kernel", default=None)
a = ap.parse_args()
cmd = ["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"]
if a.kernel:
    cmd += ["-k", a.kernel]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], [r for r in rows[2:] if len(r) == len(rows[1])]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ix = {h: hdr.index(h) for h in hdr}
num = lambda r, h: float(r[ix[h]] or 0)
tot = {h: sum(num(r, h) for r in data) for h in reasons}
allS = sum(tot.values())
print(f"{rows[0][1] if len(rows[0]) > 1 else ''}\nsamples {allS:.0f}")
for h, v in sorted(tot.items(), key=lambda t: -t[1]):
    if v > 0.005 * allS:
        print(f"  {h:28s} {100 * v / allS:5.1f}%")
# per-opcode class totals
by_op = {}
for r in data:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    op = op.split(".")[0]
    by_op[op] = by_op.get(op, 0) + num(r, "Warp Stall Sampling (All Samples)")
print("samples by opcode:", ", ".join(f"{k} {100 * v / allS:.1f}%" for k, v in sorted(by_op.items(), key=lambda t: -t[1])[:10]))
top = sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[: a.top]
for r in top:
    rs = sorted(((num(r, h), h[6:]) for h in reasons), reverse=True)[:3]
    print(f"{r[ix['Address']][-5:]} {r[ix['Source']][:52]:52s} {num(r, 'Warp Stall Sampling (All Samples)'):7.0f} "
          + " ".join(f"{n}={v:.0f}" for v, n in rs if v > 0))
