#!/bin/bash
# ncu launch list of exactly one timed bench step (run on the GPU box via gpurun,
# one GPU, after the same command exited 0 without ncu). Per-launch times are
# cold-cache and serialised: compare the kernels' shares of the step.
set -e
OUT=${1:-gpurun_out}
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > $OUT/ncu_plain.log 2>&1
ECOSERVE_NCU_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size \
    --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
