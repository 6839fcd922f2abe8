# round 2 (b): new edge/torch-op tests; ncu source-level captures of the fused quantization at
# n >= 8192 and of the transform's exchange (bank conflicts); DRAM traffic of every quant launch;
# c2/c4 bench lines with timed regions long enough for clock samples
set -x
O=gpurun_out/r02_b
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_gpu_torch_ops.py -q -x > $O/pytest_new.txt 2>&1; echo "rc=$?" >> $O/pytest_new.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fwht_rows -s 6 -c 6 -o $O/quant_big \
  python tools/ncu_quant.py 8192,16384,32768 e4m3 > $O/ncu_quant_big.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fwht_rows -s 2 -c 2 -o $O/xform_1024 \
  python tools/ncu_one.py 1024 f16,bf16 > $O/ncu_xform.log 2>&1
for q in e4m3 int8 int4; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:fwht -s 18 -c 18 --csv python tools/ncu_quant.py 128,256,512,1024,2048,4096,8192,16384,32768 $q > $O/traffic_$q.csv 2> $O/traffic_$q.err
done
timeout 300 python bench.py --workload c2 --steps 3000 --no-e2e > $O/c2.json 2> $O/c2.err
timeout 300 python bench.py --workload c4 --steps 3000 --no-e2e > $O/c4.json 2> $O/c4.err
