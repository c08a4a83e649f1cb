# 8B decode + bench: this build vs libecoserve_base.so (previous HEAD), alternating in one session
mkdir -p gpurun_out
o2=gpurun_out/ab_base.jsonl; : > $o2
for i in 1 2 3; do
  echo "== new" >> $o2; timeout 300 python tools/decode_ablate.py --one >> $o2 2>&1
  echo "== base" >> $o2; ECOSERVE_LIB_AB=paper_2504_18154_b200/libecoserve_base.so timeout 300 python tools/decode_ablate.py --one >> $o2 2>&1
done
cat $o2
