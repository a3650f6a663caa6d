"""profiles/traffic.json entry from an ncu --set full report: DRAM bytes (read + write)
per launch of the named kernel.  usage: traffic_from_ncu.py REPORT KEY KERNEL_REGEX"""
import csv, io, json, os, re, subprocess, sys

rep, key, pat = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
best = None
for row in rows[2:]:
    d = dict(zip(hdr, row))
    u = dict(zip(hdr, units))
    if not re.search(pat, d.get("Kernel Name", "")):
        continue
    b = sum(float(d[k]) * scale[u[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    best = {"dram_bytes_per_launch": b, "kernel": d["Kernel Name"], "grid": d.get("launch__grid_size"),
            "duration_ms_under_ncu": float(d["gpu__time_duration.sum"]) * (1e-3 if u["gpu__time_duration.sum"] == "us" else 1e-6 if u["gpu__time_duration.sum"] == "ns" else 1.0),
            "source": os.path.basename(rep)}
path = os.environ.get("TRAFFIC_JSON") or os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
db = json.load(open(path)) if os.path.exists(path) else {}
db[key] = best
json.dump(db, open(path, "w"), indent=1)
print(key, best)
