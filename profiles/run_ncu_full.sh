#!/bin/bash
# --set full captures of the four kernel classes of the bench step (run via gpurun on one
# GPU, after the plain command exited 0). Same one-step profiler range as run_ncu.sh.
OUT=${1:-gpurun_out}
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > $OUT/ncu_plain.log 2>&1 || exit 1
F="--set full --clock-control none --import-source on --profile-from-start off"
export ECOSERVE_NCU_RANGE=1
ncu $F -k regex:gemm_tc2_kernel -s 2 -c 1 -o $OUT/prof_gemm_prefill $CMD > $OUT/ncu_full_gp.log 2>&1
ncu $F -k regex:attn_prefill_tc_kernel -s 2 -c 1 -o $OUT/prof_attn_prefill $CMD > $OUT/ncu_full_ap.log 2>&1
ncu $F -k regex:gemm_tc_kernel -s 300 -c 4 -o $OUT/prof_gemm_decode $CMD > $OUT/ncu_full_gd.log 2>&1
ncu $F -k regex:attn_decode_kernel -s 40 -c 1 -o $OUT/prof_attn_decode $CMD > $OUT/ncu_full_ad.log 2>&1
