#!/bin/bash
# run slab_perf.py CFG SWEEPS for each library variant: tools/variants.sh CFG SWEEPS LOG name [name ...] ("base" = default lib)
cfg=$1; sw=$2; log=$3; shift 3
for v in "$@"; do
  echo "== $v" >> $log
  if [ "$v" = base ]; then
    timeout -s KILL 120 python tools/slab_perf.py $cfg $sw $v: >> $log 2>&1
  else
    ASY_LIB_VARIANT=$v timeout -s KILL 120 python tools/slab_perf.py $cfg $sw $v: >> $log 2>&1
  fi
done
