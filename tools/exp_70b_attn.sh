# 70B rank shard (TP=1 floor): decode attention split / stream-K variants
mkdir -p gpurun_out
o=gpurun_out/exp_70b_attn.jsonl; : > $o
for v in "" "ECOSERVE_ATTN_SPLITS=2" "ECOSERVE_ATTN_SPLITS=3" "ECOSERVE_ATTN_SK=1"; do
  echo "== $v" >> $o
  env $v timeout 900 python tools/tp_bench.py --tp1 --reps 2 >> $o 2>> gpurun_out/exp_70b_attn.err
done
cat $o
