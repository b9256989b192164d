"""Summarise an `ncu --set full` report (read here, no GPU) into profiles/*.json + a table:
per launch duration, DRAM bytes, tensor-pipe and DRAM utilisation, achieved TFLOP/s or GB/s."""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__grid_size", "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second"]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
idx = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3, "%": 1, "": 1, "Ghz": 1e9, "hz": 1, "Mhz": 1e6,
         "cycle/second": 1, "cycle/nsecond": 1e9, "cycle/usecond": 1e6}
recs = []
for r in rows[2:]:
    rec = {"kernel": r[idx["Kernel Name"]].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")}
    for m in metrics:
        if m in idx:
            u = units[idx[m]]
            try:
                rec[m] = float(r[idx[m]].replace(",", "")) * scale.get(u, 1)
            except ValueError:
                rec[m] = r[idx[m]]
    rec["time_us"] = rec["gpu__time_duration.sum"] * 1e6
    rec["dram_bytes"] = rec["dram__bytes_read.sum"] + rec["dram__bytes_write.sum"]
    recs.append(rec)
json.dump(recs, open(out, "w"), indent=1)
print(f"{'kernel':45s} {'us':>8s} {'DRAM MB':>8s} {'tensor%':>8s} {'dram%':>6s} {'SM GHz':>6s}")
for r in recs:
    print(f"{r['kernel'][:45]:45s} {r['time_us']:8.1f} {r['dram_bytes'] / 1e6:8.1f} "
          f"{r.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 0):8.1f} "
          f"{r.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):6.1f} "
          f"{r.get('sm__cycles_elapsed.avg.per_second', 0) / 1e9:6.2f}")
