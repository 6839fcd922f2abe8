O=gpurun_out/r02_u
mkdir -p $O
cp build/tcab/eg2a.so paper_2412_08832_b200/libhadacore.so
timeout 60 python tools/pp_probe.py > $O/quick.txt 2>&1; echo "quick rc=$?"
timeout 200 python -m pytest tests/test_gpu_quant.py -q -x -k "16384 or 32768" 2>&1 | tail -1
ROUNDS=2 bash tools/ab_so.sh "--workload quant-e4m3 --ns 16384,32768" build/tcab/eg1.so build/tcab/eg2a.so build/tcab/eg2b.so build/tcab/eg2c.so > $O/ab.txt 2>&1
ROUNDS=1 bash tools/ab_so.sh "--workload quant-int4 --ns 16384,32768" build/tcab/eg1.so build/tcab/eg2a.so build/tcab/eg2b.so build/tcab/eg2c.so >> $O/ab.txt 2>&1
cat $O/ab.txt
