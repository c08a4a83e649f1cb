for i in 1 2; do
timeout 900 python tools/tp_bench.py --tp1 --reps 2
ECOSERVE_GU_SK=0 timeout 900 python tools/tp_bench.py --tp1 --reps 2
done
