"""Per-CUDA-source-line warp-stall samples from an ncu report (needs -lineinfo + --import-source)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, hdr, agg, tot = None, None, [], 0.0
stall_cols = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
        continue
    if hdr and r[0].isdigit():
        def f(x):
            try:
                return float(x)
            except ValueError:
                return 0.0
        s = f(r[4])
        tot += s
        det = sorted(((hdr[i][6:], f(r[i])) for i in stall_cols if i < len(r) and f(r[i]) > 0),
                     key=lambda kv: -kv[1])[:3]
        agg.append((s, cur, int(r[0]), r[1].strip()[:70], det))
agg.sort(key=lambda x: -x[0])
print(f"total samples {tot:.0f}")
for s, f, ln, src, det in agg[:top]:
    print(f"{100*s/tot:5.1f}% {f}:{ln:<4d} {src:70s} " + " ".join(f"{k}={v:.0f}" for k, v in det))
