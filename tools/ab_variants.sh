#!/bin/bash
# A/B the built library variants in paper_1701_04900_b200/lib/variants on config $1
cfg=${1:-1}
cp paper_1701_04900_b200/lib/libasyflexa.so /tmp/lib_main.so
for v in paper_1701_04900_b200/lib/variants/*.so; do
  cp $v paper_1701_04900_b200/lib/libasyflexa.so
  echo "== $v" >> gpurun_out/ab.log
  timeout -s KILL 60 python tools/try_geom.py $cfg 0 0 20 >> gpurun_out/ab.log 2>&1 || echo "rc=$?" >> gpurun_out/ab.log
done
cp /tmp/lib_main.so paper_1701_04900_b200/lib/libasyflexa.so
