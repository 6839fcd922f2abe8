# round 2 (r): SIMT ablation on the current code: packed FADD2/FFMA2 shuffle
# butterflies (V-B) at the product launch table and at 2-3 CTAs per SM, the round-1 scalar form,
# vs the mma.sync product; paired step-by-step (tools/tune.py run), then ncu of the best SIMT build
set -x
O=gpurun_out/r02_r
mkdir -p $O
timeout 1200 python tools/tune.py run > $O/simt_ab.txt 2>&1
cat $O/simt_ab.txt
