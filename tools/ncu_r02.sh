#!/bin/bash
# ncu evidence for the round-2 bench line: one `--set full` capture of the update kernel per
# config (the launch shape bench.py times: CHECK sweeps per launch, cyclic schedule), summarised
# on the GPU box (traffic.json entries, metric + stall summaries), and the gpu__time_duration
# launch list of the default bench command.  Reports are kept in /tmp (too large to copy back).
K='regex:dense_async_kernel|dense_slabt_kernel|sparse_async_kernel'
mkdir -p /tmp/ncu
for cs in "1 5" "2 25" "3 1" "4 500"; do
  set -- $cs
  timeout 600 ncu --set full --clock-control none --import-source on -k "$K" -c 1 -f -o /tmp/ncu/r02_c$1 \
    python tools/slab_one.py $1 $2 cyclic > gpurun_out/r02_c$1.log 2>&1
  python tools/ncu_traffic.py /tmp/ncu/r02_c$1.ncu-rep $1 $2 "profiles/r02_ncu_c$1.txt (ncu --set full, one launch of $2 sweeps of configs[$1], cyclic)" >> gpurun_out/r02_c$1.log 2>&1
  fn=$(ncu -i /tmp/ncu/r02_c$1.ncu-rep --page raw --csv --print-kernel-base mangled 2>/dev/null | python -c "import csv,sys; r=list(csv.reader(sys.stdin)); print(r[2][r[0].index('Kernel Name')] if 'Kernel Name' in r[0] else '')")
  python tools/ncu_summary.py /tmp/ncu/r02_c$1.ncu-rep "$fn" "configs[$1]: ncu --set full, one launch of $2 sweeps (cyclic)" > gpurun_out/r02_ncu_c$1.txt 2>&1
done
cp profiles/traffic.json gpurun_out/traffic.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02_launches_bench.log 2>&1
