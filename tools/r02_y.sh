O=gpurun_out/r02_y
mkdir -p $O
cp build/f32ab/p24g3.so paper_2412_08832_b200/libhadacore.so
timeout 60 python tools/f32_mc_check.py > $O/check.txt 2>&1; echo "check rc=$?"; cat $O/check.txt
ROUNDS=2 bash tools/ab_so.sh "--workload f32 --ns 32768" build/f32ab/p16g2.so build/f32ab/p24g3.so build/f32ab/p8g2.so > $O/ab.txt 2>&1
cat $O/ab.txt
