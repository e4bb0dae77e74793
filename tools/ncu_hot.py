"""Print the hottest SASS instructions (warp-stall samples) of an ncu report,
with the nearest preceding CUDA source line (needs -lineinfo + --import-source)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"]
                     + (["-k", f"regex:{kern}"] if kern else []), capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks, cur = [], None
for r in rows:
    if len(r) >= 2 and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
        continue
    if cur is None:
        continue
    if r and r[0] == "Address":
        cur["hdr"] = r
        continue
    cur["rows"].append(r)
for b in blocks[:1]:
    h = b["hdr"]
    si = h.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in b["rows"]:
        if len(r) > si:
            try:
                data.append((int(r[si] or 0), r))
            except ValueError:
                pass
    tot = sum(x for x, _ in data) or 1
    print(b["name"], "samples", tot)
    for x, r in sorted(data, key=lambda t: -t[0])[:top]:
        print(f"{x:6d} {100 * x / tot:5.1f}%  {r[1][:100]}")
