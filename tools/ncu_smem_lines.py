"""Per-source-line shared-memory excess wavefronts (bank conflicts) and stall samples of ONE kernel
result in an ncu report. Usage: ncu_smem_lines.py report.ncu-rep [launch_skip] [top]."""
import csv, subprocess, sys
rep = sys.argv[1]
skip = sys.argv[2] if len(sys.argv) > 2 else "0"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-skip", skip,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
hdr, cur, rows = None, None, []
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Name":
        cur = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
    elif hdr and r[0].isdigit():
        def g(k):
            try:
                return float(r[hdr[k]])
            except (KeyError, IndexError, ValueError):
                return 0.0
        rows.append((cur, int(r[0]), r[1].strip()[:80], g("Warp Stall Sampling (All Samples)"),
                     g("L1 Wavefronts Shared"), g("L1 Wavefronts Shared Excessive")))
tot_s = sum(x[3] for x in rows) or 1
tot_w = sum(x[4] for x in rows) or 1
print(f"samples {tot_s:.0f}  shared wavefronts {tot_w:.3g}  excessive {sum(x[5] for x in rows):.3g}")
for f, ln, src, s, w, e in sorted(rows, key=lambda x: -(x[4] + x[3] * 1e3))[:top]:
    print(f"{100*s/tot_s:5.1f}% smp  wf {w:10.3g} exc {e:10.3g}  {f}:{ln:<4d} {src}")
