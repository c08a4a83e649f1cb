# final round-2 evidence at HEAD on one B200: bench, ncu launch list, --set full captures
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 900 bash profiles/run_ncu.sh gpurun_out
timeout 1800 bash profiles/run_ncu_full.sh gpurun_out
for f in gpurun_out/prof_*.ncu-rep; do
  ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null
done
ls -la gpurun_out; cat gpurun_out/final_bench.json
