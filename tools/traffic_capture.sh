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
# C3 FULL: 30-shot steps as two 15-shot chains (forward + history store,
# three-level adjoint + imaging); skip the warm-up launches
ncu --replay-mode application --cache-control none --clock-control none --metrics $M \
    -k regex:k_step --launch-count 400 --csv \
    python tools/profile_step.py --config c3 --reps 40 > "$OUT/traffic_c3.csv" 2> "$OUT/traffic_c3.err"
# C5 BOUNDARY: 8-shot steps (band-storing forward, fused reverse + adjoint)
ncu --replay-mode application --cache-control none --clock-control none --metrics $M \
    -k regex:k_step --launch-count 400 --csv \
    python tools/profile_step.py --config c5 --recon boundary --shots 8 --nt 400 --reps 40 \
    > "$OUT/traffic_c5.csv" 2> "$OUT/traffic_c5.err"
