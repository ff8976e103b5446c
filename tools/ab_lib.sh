#!/bin/bash
# Interleaved A/B of the default bench workload against variant arms:
# alternating processes, ms per C3 gradient and step-kernel times.
#   bash tools/ab_lib.sh ROUNDS "ENV=VAL ..." ["ENV=VAL ..." ...]
# e.g. bash tools/ab_lib.sh 3 "SG_LIB=var/lib_variant.so" "SG_GROUP=6"
R=$1; shift
for i in $(seq 1 $R); do
  for arm in "" "$@"; do
    env $arm python bench.py --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d.get('roofline',{})
print('[${arm:-default}]', round(d['ms_per_step'],2), 'fwd', round(1e3*r.get('forward_ms_per_step',0),2), 'adj', round(1e3*r.get('adjoint_ms_per_step',0),2), d['clocks']['sm_mhz'])"
  done
done
