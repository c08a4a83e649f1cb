# full GPU suite + one bench line (run under gpurun)
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/full_tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err
tail -5 gpurun_out/full_tests.txt; cat gpurun_out/full_bench.json
