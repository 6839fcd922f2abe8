set -x
O=gpurun_out/r02_s
mkdir -p $O
cp build/tune/libhc_simt_c3.so paper_2412_08832_b200/libhadacore.so
timeout 600 ncu --set full --clock-control none -k regex:fwht -s 3 -c 3 -o $O/simt_c3 python tools/ncu_one.py 256,4096,32768 f16 > $O/ncu_simt.log 2>&1
cp build/tune/libhc_tuned.so paper_2412_08832_b200/libhadacore.so
timeout 600 ncu --set full --clock-control none -k regex:fwht -s 3 -c 3 -o $O/mma python tools/ncu_one.py 256,4096,32768 f16 > $O/ncu_mma.log 2>&1
