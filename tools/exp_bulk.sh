# bulk-copy epilogue copy-out: decode GEMM parity + 8B decode / 70B shard A/B against libecoserve_base.so
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_ops.py -k "gemm" 2>&1 | tail -3 > gpurun_out/bulk_ops.txt
timeout 900 python -m pytest -q -x tests/test_gpu_instance.py tests/test_gpu_fullsize.py -k "not variants" 2>&1 | tail -3 >> gpurun_out/bulk_ops.txt
o=gpurun_out/exp_bulk.jsonl; : > $o
for i in 1 2 3; do
  echo "== new" >> $o; timeout 300 python tools/decode_ablate.py --one >> $o 2>&1
  echo "== base" >> $o; ECOSERVE_LIB_AB=paper_2504_18154_b200/libecoserve_base.so timeout 300 python tools/decode_ablate.py --one >> $o 2>&1
done
for i in 1 2; do
  echo "== new 70b" >> $o; timeout 900 python tools/tp_bench.py --tp1 --reps 2 >> $o 2>&1
  echo "== base 70b" >> $o; ECOSERVE_LIB_AB=paper_2504_18154_b200/libecoserve_base.so timeout 900 python tools/tp_bench.py --tp1 --reps 2 >> $o 2>&1
done
cat gpurun_out/bulk_ops.txt $o
