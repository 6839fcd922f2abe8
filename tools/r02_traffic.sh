# per-launch DRAM traffic JSONs (bench.py roofline.traffic) on the final build: quant sweeps + fp32 sweep
O=gpurun_out/r02_traffic
mkdir -p $O
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for q in e4m3 int8 int4; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:fwht -s 18 -c 18 --csv --log-file $O/quant-$q.csv \
    python tools/ncu_quant.py 128,256,512,1024,2048,4096,8192,16384,32768 $q > /dev/null 2>&1; echo "$q rc=$?"
done
timeout 600 ncu --metrics $M --clock-control none -k regex:fwht -s 15 -c 15 --csv --log-file $O/f32.csv \
  python tools/ncu_one.py 2,4,8,16,32,64,128,256,512,1024,2048,4096,8192,16384,32768 f32 > /dev/null 2>&1; echo "f32 rc=$?"
