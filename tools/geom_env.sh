#!/bin/bash
# run try_geom with several (RPL, NS) env overrides: args: cfg sweeps "rpl:ns" ...
cfg=$1; sw=$2; shift 2
for v in "$@"; do
  r=${v%%:*}; n=${v##*:}
  echo -n "RPL=$r NS=$n: " >> gpurun_out/genv.log
  ASY_DENSE_RPL=$r ASY_DENSE_NS=$n timeout -s KILL 60 python tools/try_geom.py $cfg 0 0 $sw >> gpurun_out/genv.log 2>&1 || echo "rc=$?" >> gpurun_out/genv.log
done
