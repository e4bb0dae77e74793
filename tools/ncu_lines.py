"""Warp-stall samples per CUDA source line of an ncu report (needs -lineinfo):
    python tools/ncu_lines.py report.ncu-rep [top] [kernel-regex]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kern = sys.argv[3] if len(sys.argv) > 3 else ""
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"]
if kern:
    cmd += ["-k", f"regex:{kern}"]
rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
fname, hdr, out = "", None, []
for r in rows:
    if len(r) == 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit() and r[2] == "-":  # source-line aggregate
        d = dict(zip(hdr[4:], r[4:]))
        d["Source"] = r[1]
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        if s:
            reasons = {k[6:]: int(v) for k, v in d.items()
                       if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v)}
            top3 = sorted(reasons.items(), key=lambda kv: -kv[1])[:3]
            out.append((s, fname, r[0], d["Source"].strip()[:70], top3))
tot = sum(o[0] for o in out) or 1
for s, f, ln, src, t3 in sorted(out, key=lambda o: -o[0])[:top]:
    print(f"{s:7d} {100 * s / tot:5.1f}% {f}:{ln:5s} {src:70s} {t3}")
