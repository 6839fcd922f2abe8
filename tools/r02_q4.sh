O=gpurun_out/r02_q4
mkdir -p $O
ROUNDS=2 bash tools/ab_so.sh "--workload quant-int4 --ns 512,1024,2048" build/q4/base.so build/q4/a.so build/q4/b.so build/q4/c.so build/q4/d.so build/q4/e.so > $O/ab.txt 2>&1
cat $O/ab.txt
