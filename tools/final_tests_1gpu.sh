# the driver's round-end checks on one GPU: pytest -m gpu (with durations) and smoke()
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -x -q --durations=30 2>&1 | tail -60 > gpurun_out/tests_1gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
tail -45 gpurun_out/tests_1gpu.txt; cat gpurun_out/smoke.txt
