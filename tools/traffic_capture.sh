#!/bin/bash
# Steady-state DRAM bytes of the shipped step kernels (run on the GPU box):
# ncu application replay with --cache-control none, so every profiled launch
# sees the L2 state the preceding launches of the real launch sequence left
# (the --set full captures flush caches per replay: cold-cache upper bounds).
#   bash tools/traffic_capture.sh OUTDIR
set -e
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum
NCU="ncu --replay-mode application --cache-control none --clock-control none --metrics $M --csv"
# C3 FULL, inside one real gradient (no graphs: 2 chains x 4000 forward
# launches, then 2 x 4000 adjoint launches): the history planes stream to and
# from HBM as in the bench.  Launches 3000..3399 are forward steps, 11000..
# 11399 adjoint steps.
$NCU -k regex:k_step --launch-skip 3000 --launch-count 400 \
    python tools/one_gradient.py --config c3 > "$OUT/traffic_c3_fwd.csv" 2> "$OUT/traffic_c3_fwd.err"
$NCU -k regex:k_step --launch-skip 11000 --launch-count 400 \
    python tools/one_gradient.py --config c3 > "$OUT/traffic_c3_adj.csv" 2> "$OUT/traffic_c3_adj.err"
# C5 BOUNDARY: 14-shot steps (the batch a full C5 gradient runs: two 7-shot chains) (band-storing forward, fused reverse + adjoint);
# the band store walks a new slot per launch, the fields are far larger than L2
$NCU -k regex:k_step --launch-count 400 \
    python tools/profile_step.py --config c5 --recon boundary --shots 14 --nt 400 --reps 40 \
    > "$OUT/traffic_c5.csv" 2> "$OUT/traffic_c5.err"
