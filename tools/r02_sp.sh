O=gpurun_out/r02_sp
mkdir -p $O
timeout 60 python tools/pp_probe.py > $O/quick.txt 2>&1; echo "quick rc=$?"
timeout 300 python -m pytest tests/test_gpu_quant.py tests/test_gpu_jitter.py -q -x -k "4096 or 8192 or 16384 or 32768 or jitter" 2>&1 | tail -1
ROUNDS=2 bash tools/ab_so.sh "--workload quant-e4m3 --ns 16384,32768" build/tcab/cur.so build/tcab/split.so > $O/ab.txt 2>&1
ROUNDS=1 bash tools/ab_so.sh "--workload quant-int4 --ns 4096,8192,16384,32768" build/tcab/cur.so build/tcab/split.so >> $O/ab.txt 2>&1
cat $O/ab.txt
cp build/tcab/split.so paper_2412_08832_b200/libhadacore.so
