"""DRAM traffic per sweep of the update kernel from an `ncu --set full` report of one launch,
written into profiles/traffic.json (the bench line's roofline.traffic, per config and kernel).
usage: python tools/ncu_traffic.py REPORT.ncu-rep CONFIG_IDX SWEEPS_IN_THE_LAUNCH SOURCE_TXT"""
import csv
import io
import json
import os
import subprocess
import sys

rep, idx, sweeps, src = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))
units = dict(zip(h, u))


def val(k):
    x = float(d[k].replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(units[k], 1)


kernel = d["Kernel Name"].split("(")[0].split("<")[0].strip()
kernel = kernel.replace("void ", "")
if not kernel.startswith("asy::"):
    kernel = "asy::" + kernel
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "traffic.json")
t = json.load(open(path)) if os.path.exists(path) else {}
t = {k: w for k, w in t.items() if k.startswith("configs[")}
t[f"configs[{idx}]"] = {"kernel": kernel, "dram_read_bytes_per_sweep": val("dram__bytes_read.sum") / sweeps,
                        "dram_write_bytes_per_sweep": val("dram__bytes_write.sum") / sweeps,
                        "kernel_ms_per_sweep_under_ncu": float(d["gpu__time_duration.sum"].replace(",", "")) / sweeps,
                        "sweeps_in_launch": sweeps, "source": src}
json.dump(t, open(path, "w"), indent=1)
print(json.dumps(t[f"configs[{idx}]"]))
