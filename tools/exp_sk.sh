# balanced split-K decode projections (ECOSERVE_DEC_SK=1) and auto stream-K attention: parity + A/B
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_ops.py -k "balanced or gemm_decode or attention_decode" 2>&1 | tail -3 > gpurun_out/sk_ops.txt
o=gpurun_out/exp_sk.jsonl; : > $o
for i in 1 2; do
  for v in "ECOSERVE_DEC_SK=0" "ECOSERVE_DEC_SK=1"; do
    echo "== 8b $v" >> $o
    env $v timeout 300 python tools/decode_ablate.py --one >> $o 2>> gpurun_out/exp_sk.err
  done
done
for v in "ECOSERVE_DEC_SK=0" "ECOSERVE_DEC_SK=1" "ECOSERVE_DEC_SK=1 ECOSERVE_ATTN_SK=0"; do
  echo "== 70b shard $v" >> $o
  env $v timeout 900 python tools/tp_bench.py --tp1 --reps 2 >> $o 2>> gpurun_out/exp_sk.err
done
cat gpurun_out/sk_ops.txt $o
