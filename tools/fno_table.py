"""Format an `ncu --csv --metrics ...` capture of tools/run_fno.py (two forwards) as the per-kernel
table of the second forward (profiles/r1_k5_fno_kernels_v*.txt)."""
import csv, sys
SCALE = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "%": 1.0}
data, hdr = {}, None
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        data.setdefault(int(d["ID"]), [d["Kernel Name"], {}])[1][d["Metric Name"]] = v
ids = sorted(data)
casts = [i for i in ids if "cast_f64_to_f32" in data[i][0]]
ids = [i for i in ids if i >= casts[-1] and not data[i][0].startswith("void at::")]
print("C5 FNO forward (4096 x 1024, width 64, 16 modes, 4 layers): ncu --metrics, --clock-control none (cold caches,")
print("serialised launches), second of two forwards. TB/s = (DRAM read + write) / time.")
print(f"{'kernel':52s} {'time us':>8s} {'rd GB':>7s} {'wr GB':>7s} {'TB/s':>6s} {'issue%':>7s} {'tensor%':>8s} {'fma%':>6s}")
tot = 0.0
for i in ids:
    n, m = data[i]
    t = m["gpu__time_duration.sum"]
    rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
    tot += t
    print(f"{n[:52]:52s} {t:8.1f} {rd:7.3f} {wr:7.3f} {(rd + wr) / t * 1e3:6.2f} "
          f"{m['smsp__issue_active.avg.pct_of_peak_sustained_active']:7.1f} "
          f"{m['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed']:8.1f} "
          f"{m['sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active']:6.1f}")
print(f"{'total':52s} {tot:8.1f}")
