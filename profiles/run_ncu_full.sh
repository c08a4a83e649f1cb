#!/bin/bash
# --set full captures of the two GEMM flavours (run via gpurun on one GPU, after a plain run).
OUT=${1:-gpurun_out}
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > $OUT/ncu_plain.log 2>&1 || exit 1
# gemm launches: ~1548 in the setup prefill, then the first warmup step's prefill (129), then decode
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1560 -c 2 \
    -o $OUT/prof_gemm_prefill $CMD > $OUT/ncu_full_gp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1700 -c 4 \
    -o $OUT/prof_gemm_decode $CMD > $OUT/ncu_full_gd.log 2>&1
