# 70B TP=2 decode at SURVEY 8(d)'s worked point (B = 128, c = 600) and the rank shard alone
mkdir -p gpurun_out
o=gpurun_out/tp_c600.jsonl; : > $o
timeout 1200 python tools/tp_bench.py --reps 2 --prompt 600 >> $o 2>> gpurun_out/tp_c600.err
timeout 1200 python tools/tp_bench.py --reps 2 --prompt 600 --tp1 >> $o 2>> gpurun_out/tp_c600.err
cat $o
