#!/bin/bash
# One ncu --set full capture per shipped step kernel (run on the GPU box, one
# GPU, after the same commands exited 0 without ncu):
#   bash tools/ncu_full_capture.sh OUTDIR
# tools/profile_step.py --reps 2 launches, per chain and in this order: 2
# warm-up + 2 timed forward steps, then 2 + 2 adjoint steps (two chains: 8
# forward launches, then 8 adjoint launches).  Summaries: tools/ncu_summary.py.
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
NCU="ncu --set full --clock-control none --import-source on -k regex:k_step"
$NCU -s 4 -c 2 -f -o "$OUT/ncu_fwd_c3" python tools/profile_step.py --config c3 --reps 2 > "$OUT/ncu_fwd_c3.log" 2>&1
$NCU -s 12 -c 2 -f -o "$OUT/ncu_adj_c3" python tools/profile_step.py --config c3 --reps 2 > "$OUT/ncu_adj_c3.log" 2>&1
$NCU -s 4 -c 2 -f -o "$OUT/ncu_fwd_c5" python tools/profile_step.py --config c5 --recon boundary --shots 8 --nt 400 --reps 2 > "$OUT/ncu_fwd_c5.log" 2>&1
$NCU -s 12 -c 2 -f -o "$OUT/ncu_adj_c5" python tools/profile_step.py --config c5 --recon boundary --shots 8 --nt 400 --reps 2 > "$OUT/ncu_adj_c5.log" 2>&1
# summaries on the box (the reports are ~20 MB each with sources; gpurun
# brings back at most 64 MiB): key metrics, and the hottest source lines
for r in fwd_c3 adj_c3 fwd_c5 adj_c5; do
  python tools/ncu_summary.py "$OUT/ncu_$r.ncu-rep" > "$OUT/ncu_$r.txt" 2>&1
  ncu -i "$OUT/ncu_$r.ncu-rep" --page source --csv --print-source cuda 2>/dev/null \
      | python tools/ncu_hot_lines.py > "$OUT/ncu_${r}_hot_lines.txt" 2>&1
  case " ${KEEP_REP:-} " in *" $r "*) ;; *) rm -f "$OUT/ncu_$r.ncu-rep" ;; esac
done
ls -la "$OUT"
