"""Write a text summary of an `ncu --set full` report (metrics + hottest source lines).
usage: python tools/ncu_summary.py REPORT.ncu-rep KERNEL_MANGLED_NAME TITLE > profiles/<name>.txt
Needs the library the report was taken with (lineinfo) at paper_1701_04900_b200/lib/libasyflexa.so."""
import csv
import io
import os
import subprocess
import sys
import tempfile

rep, fn, title = sys.argv[1], sys.argv[2], sys.argv[3]
HERE = os.path.dirname(os.path.abspath(__file__))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
print(f"# {title}")
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
        "lts__t_requests_srcunit_tex_op_red.sum", "smsp__average_warp_latency_issue_stalled_no_instruction"]
for w in want:
    if w in h:
        i = h.index(w)
        print(f"{w:60s} {v[i]:>16s} {u[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
with tempfile.TemporaryDirectory() as d:
    open(os.path.join(d, "s.csv"), "w").write(src)
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(HERE, "..", "paper_1701_04900_b200", "lib",
                                                             "libasyflexa.so")], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    g = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    open(os.path.join(d, "g.sass"), "w").write(g)
    out = subprocess.run([sys.executable, os.path.join(HERE, "ncu_lines.py"), os.path.join(d, "s.csv"),
                          os.path.join(d, "g.sass"), fn, "30"], capture_output=True, text=True).stdout
print("\n# warp-stall samples by source line (share, top stall reasons)")
print(out)
st = subprocess.run([sys.executable, os.path.join(HERE, "ncu_stalls.py"), "/dev/stdin", "0"], input=src,
                    capture_output=True, text=True).stdout
print("# stall reasons over the kernel")
print("\n".join(st.split("\n")[:2]))
