# round 2 (p): evidence for the tcgen05 fused quantization (routed build): ncu --set full of the
# n = 16384 / 32768 launches (E4M3, INT4), DRAM traffic of every quant launch, bench lines
set -x
O=gpurun_out/r02_p
mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fwht_quant_tc -s 4 -c 4 -o $O/tc_e4m3 \
  python tools/ncu_quant.py 16384,32768 e4m3 > $O/ncu_e4m3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fwht_quant_tc -s 4 -c 4 -o $O/tc_int4 \
  python tools/ncu_quant.py 16384,32768 int4 > $O/ncu_int4.log 2>&1
for q in e4m3 int8 int4; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:fwht -s 18 -c 18 --csv python tools/ncu_quant.py 128,256,512,1024,2048,4096,8192,16384,32768 $q > $O/traffic_$q.csv 2> $O/traffic_$q.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_quant_e4m3.csv \
  python bench.py --workload quant-e4m3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for q in e4m3 int8 int4; do
  timeout 300 python bench.py --workload quant-$q --no-e2e --no-cpu-baseline > $O/quant-$q.json 2> $O/quant-$q.err
done
