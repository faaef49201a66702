#!/bin/bash
cp paper_1701_04900_b200/lib/libasyflexa.so /tmp/lib_main.so
for v in paper_1701_04900_b200/lib/variants/*.so; do
  cp $v paper_1701_04900_b200/lib/libasyflexa.so
  n=$(basename $v .so)
  timeout -s KILL 60 python tools/try_geom.py ${CFG:-1} 0 0 20 > gpurun_out/ab_$n.log 2>&1
  ASY_TRACE=100000 ASY_TRACE_FILE=gpurun_out/tr_$n.bin timeout -s KILL 60 python tools/try_geom.py ${CFG:-1} 0 0 5 >> gpurun_out/ab_$n.log 2>&1
done
cp /tmp/lib_main.so paper_1701_04900_b200/lib/libasyflexa.so
