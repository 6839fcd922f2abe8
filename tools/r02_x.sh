O=gpurun_out/r02_x
mkdir -p $O
ROUNDS=2 bash tools/ab_so.sh "--workload f32 --ns 2048,4096,8192,16384" build/f32ab/base.so build/f32ab/big8k.so build/f32ab/big4k.so > $O/ab.txt 2>&1
cat $O/ab.txt
