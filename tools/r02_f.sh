# round 2 (f): where the tcgen05 fused quantization spends its time: diagnostic builds
# (HC_TC_DIAG bit 0 = no phase-A arithmetic, 1 = no epilogue, 2 = no MMAs) at n = 8192, 32768,
# then one ncu --set full capture of the default build at n = 8192 and 32768
set -x
O=gpurun_out/r02_f
mkdir -p $O
ROUNDS=1 bash tools/ab_so.sh "--workload quant-e4m3 --ns 8192,32768" build/tcdiag/d0.so build/tcdiag/d1.so build/tcdiag/d2.so build/tcdiag/d4.so build/tcdiag/d3.so > $O/diag.txt 2>&1
cat $O/diag.txt
cp build/tcdiag/d0.so paper_2412_08832_b200/libhadacore.so
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fwht_quant_tc -s 4 -c 4 -o $O/tc \
  python tools/ncu_quant.py 8192,32768 e4m3 > $O/ncu.log 2>&1
tail -3 $O/ncu.log
