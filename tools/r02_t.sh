# round 2 (t): fp32 n = 2^15 top-bit-first multicast kernel: parity + jitter tests, A/B vs the pair kernel
set -x
O=gpurun_out/r02_t
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_f32.py tests/test_gpu_jitter.py -q -x > $O/pytest_f32.txt 2>&1; echo "rc=$?" >> $O/pytest_f32.txt
tail -3 $O/pytest_f32.txt
ROUNDS=2 bash tools/ab_so.sh "--workload f32 --ns 16384,32768" build/f32ab/pair.so build/f32ab/mc.so > $O/ab.txt 2>&1
cat $O/ab.txt
cp build/f32ab/mc.so paper_2412_08832_b200/libhadacore.so
