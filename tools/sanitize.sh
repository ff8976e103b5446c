#!/bin/bash
# compute-sanitizer runs of the small 60 x 40 case (run on the GPU box):
#   bash tools/sanitize.sh OUTDIR
# racecheck (shared-memory hazards of the TMA/mbarrier rings), synccheck
# (barrier misuse), memcheck (out-of-bounds / misaligned), initcheck (reads of
# uninitialised device memory).  Each log ends with the tool's ERROR SUMMARY.
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
CS=${CS:-/usr/local/cuda/bin/compute-sanitizer}
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  [ "$tool" = initcheck ] && extra="--track-unused-memory no"
  timeout ${SAN_TIMEOUT:-900} $CS --tool $tool $extra --print-limit 20 \
      python tools/sanitize_case.py ${SAN_ARGS:-} > "$OUT/sanitizer_$tool.log" 2>&1
  echo "$tool rc=$?" >> "$OUT/sanitizer_$tool.log"
  grep -E "ERROR SUMMARY|rc=" "$OUT/sanitizer_$tool.log" | tail -2
done
