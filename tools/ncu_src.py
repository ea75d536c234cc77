"""Per-source-line warp-stall hot spots of one kernel in an ncu report:
    python tools/ncu_src.py REPORT.ncu-rep KERNEL_REGEX [N]
(ncu --page source --csv --print-source sass,cuda, aggregated per CUDA line)."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, data = "?", None, []
for r in rows:
    if r and r[0] in ("File Path", "File Name"):
        fname, hdr = r[1].split("/")[-1], None
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit() and len(r) == len(hdr):
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        i_e = hdr.index("Instructions Executed")
        data.append((int(r[i_s] or 0), int(r[i_e] or 0), fname, r[0], r[1]))
tot = sum(d[0] for d in data) or 1
print(f"{kern}: {tot} samples")
for s, e, f, ln, src in sorted(data, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% {e:>11} {f}:{ln}  {src.strip()[:100]}")
