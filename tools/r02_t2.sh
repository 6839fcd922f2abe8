O=gpurun_out/r02_t
mkdir -p $O
ROUNDS=1 bash tools/ab_so.sh "--workload f32 --ns 32768" build/f32ab/pair.so build/f32ab/mc_s3r2.so build/f32ab/mc_s4.so build/f32ab/mc_s5.so > $O/ab2.txt 2>&1
cat $O/ab2.txt
