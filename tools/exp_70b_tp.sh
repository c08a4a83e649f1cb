# 70B: rank shard decode attention variants (alternating A/B), TP=2 pair decode with profile
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_ops.py -k "stream_k" 2>&1 | tail -3 > gpurun_out/sk_attn_ops.txt
o=gpurun_out/exp_70b_tp.jsonl; : > $o
for i in 1 2; do
  for v in "ECOSERVE_ATTN_SK=0" "ECOSERVE_ATTN_SK=1" "ECOSERVE_ATTN_STAGES=2"; do
    echo "== 70b shard $v" >> $o
    env $v timeout 900 python tools/tp_bench.py --tp1 --reps 2 >> $o 2>> gpurun_out/exp_70b_tp.err
  done
done
for v in "ECOSERVE_ATTN_SK=0" "ECOSERVE_ATTN_SK=1"; do
  echo "== 70b TP=2 $v" >> $o
  env $v timeout 1200 python tools/tp_bench.py --reps 2 >> $o 2>> gpurun_out/exp_70b_tp.err
done
echo "== 70b TP=2 profile" >> $o
timeout 1200 python tools/tp_bench.py --reps 1 --profile >> $o 2>> gpurun_out/exp_70b_tp.err
cat gpurun_out/sk_attn_ops.txt $o
# 8B decode: this build vs libecoserve_base.so (previous HEAD), alternating
o2=gpurun_out/ab_base.jsonl; : > $o2
for i in 1 2 3; do
  echo "== new" >> $o2; timeout 300 python tools/decode_ablate.py --one >> $o2 2>&1
  echo "== base" >> $o2; ECOSERVE_LIB_AB=paper_2504_18154_b200/libecoserve_base.so timeout 300 python tools/decode_ablate.py --one >> $o2 2>&1
done
cat $o2
