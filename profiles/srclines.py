#!/usr/bin/env python3
"""Top source lines (and SASS instructions) of one kernel by warp-stall
samples, from an ncu report captured with --import-source on (kernel compiled
with -lineinfo).

  python profiles/srclines.py <report.ncu-rep> <kernel-regex> [top] [--sass]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 40
sass = "--sass" in sys.argv
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
lines, instrs, fname, hdr, cur = [], [], None, None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = 4
        ii = 7
        continue
    if hdr is None or len(r) <= ii:
        continue
    try:
        samp = float(r[si]) if r[si] not in ("", "-") else 0.0
        inst = float(r[ii]) if r[ii] not in ("", "-") else 0.0
    except ValueError:
        continue
    if r[0]:
        cur = f"{fname}:{r[0]}"
        lines.append((samp, inst, cur, r[1].strip()[:80]))
    elif r[2] not in ("", "..."):
        instrs.append((samp, inst, cur, r[3].strip()[:60]))
recs = instrs if sass else lines
tot = sum(x[0] for x in recs) or 1
toti = sum(x[1] for x in recs) or 1
print(f"# {kern}: {tot:.0f} stall samples, {toti:.3e} warp instructions")
for s, i, loc, src in sorted(recs, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% smp {100 * i / toti:5.1f}% ins  {loc:22s} {src}")

if "--ops" in sys.argv:
    agg = {}
    for s_, i_, loc, src in instrs:
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        a = agg.setdefault(op, [0.0, 0.0])
        a[0] += s_
        a[1] += i_
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print(f"# by opcode: {ti:.3e} warp instructions")
    for op, (s_, i_) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
        print(f"{op:14s} {100 * i_ / ti:5.1f}% ins {100 * s_ / ts:5.1f}% smp")
