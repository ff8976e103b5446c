#!/bin/bash
# Interleaved A/B of the default bench workload against variant arms:
# alternating processes, ms per C3 gradient and step-kernel times.
#   bash tools/ab_lib.sh ROUNDS "ENV=VAL ..." ["ENV=VAL ..." ...]
# e.g. bash tools/ab_lib.sh 3 "SG_LIB=var/lib_variant.so" "SG_GROUP=6"
# AB_ARGS: extra bench.py arguments (e.g. "--config c5 --steps 1 --warmup 1")
R=$1; shift
for i in $(seq 1 $R); do
  for arm in "" "$@"; do
    env $arm python bench.py --steps 3 --warmup 3 --no-cpu --no-c5-kernels ${AB_ARGS:-} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); k=d.get('roofline',{}).get('kernels',{})
print('[${arm:-default}]', round(d['ms_per_step'],2), 'ms/gradient;', ' '.join('%s %.2f us' % (n, 1e3*v['ms_per_step']) for n,v in k.items()), d['clocks']['sm_mhz'], 'MHz')"
  done
done
