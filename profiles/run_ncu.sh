#!/bin/bash
# ncu evidence for the bench (run on the GPU box via gpurun, one GPU).
# 1) plain run of the exact command; 2) launch list (cold, serialised: compare shares);
# 3) --set full captures of the top kernels (prefill GEMM, decode GEMM, both attentions).
set -e
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
OUT=${1:-gpurun_out}
$CMD > $OUT/ncu_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 17500 -c 7000 --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:'gemm_tc_kernel<256>' -s 4 -c 3 -o $OUT/prof_gemm_prefill $CMD > $OUT/ncu_full1.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:'gemm_tc_kernel<128>' -s 200 -c 4 -o $OUT/prof_gemm_decode $CMD > $OUT/ncu_full2.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:'attn_(prefill|decode)_kernel' -s 40 -c 2 -o $OUT/prof_attn_prefill $CMD > $OUT/ncu_full3.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:'attn_decode_kernel' -s 100 -c 2 -o $OUT/prof_attn_decode $CMD > $OUT/ncu_full4.log 2>&1
