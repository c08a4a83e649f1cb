mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_edge.py -k "QKV_INKERNEL" 2>&1 | tail -3 > gpurun_out/qkvk_ops.txt
o=gpurun_out/exp_qkvk.jsonl; : > $o
for i in 1 2 3; do
  for v in "ECOSERVE_QKV_INKERNEL=0" "ECOSERVE_QKV_INKERNEL=1"; do
    echo "== 8b $v" >> $o; env $v timeout 300 python tools/decode_ablate.py --one >> $o 2>&1
  done
done
for i in 1 2; do
  for v in "ECOSERVE_QKV_INKERNEL=0" "ECOSERVE_QKV_INKERNEL=1"; do
    echo "== 70b $v" >> $o; env $v timeout 900 python tools/tp_bench.py --tp1 --reps 2 >> $o 2>&1
  done
done
cat gpurun_out/qkvk_ops.txt $o
