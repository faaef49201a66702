#!/bin/bash
# A/B the built library variants in paper_1701_04900_b200/lib/variants on the configs given
cp paper_1701_04900_b200/lib/libasyflexa.so /tmp/lib_main.so
for v in paper_1701_04900_b200/lib/variants/*.so; do
  cp $v paper_1701_04900_b200/lib/libasyflexa.so
  for cfg in "$@"; do
    echo "== $v cfg $cfg" >> gpurun_out/ab.log
    timeout -s KILL 60 python tools/try_geom.py $cfg 0 0 ${SWEEPS:-20} >> gpurun_out/ab.log 2>&1 || echo "rc=$?" >> gpurun_out/ab.log
  done
done
cp /tmp/lib_main.so paper_1701_04900_b200/lib/libasyflexa.so
