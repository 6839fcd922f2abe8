# every bench.py workload once (fresh JSON lines for profiles/), then the default line last
set -x
python -m paper_2412_08832_b200.build >/dev/null
mkdir -p gpurun_out/final
for w in c1 c5 small f32 lab qk-rotate qk-quant quant-e4m3 quant-int8 quant-int4; do
  timeout 400 python bench.py --workload $w --no-e2e --no-cpu-baseline > gpurun_out/final/$w.json 2> gpurun_out/final/$w.err
done
for q in e4m3 int8 int4; do
  timeout 300 python bench.py --workload quant-$q --ns 2,4,8,16,32,64 --no-e2e --no-cpu-baseline > gpurun_out/final/quant-$q-small.json 2>/dev/null
done
python bench.py > gpurun_out/final/fwht.json 2> gpurun_out/final/fwht.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final/reference.json 2> gpurun_out/final/reference.err
timeout 300 python bench.py --workload qk-rotate --ns 8,16,32,64 --no-e2e --no-cpu-baseline > gpurun_out/final/qk-rotate-small-n.json 2>/dev/null
timeout 300 python bench.py --workload qk-quant --ns 8,16,32,64 --no-e2e --no-cpu-baseline > gpurun_out/final/qk-quant-small-n.json 2>/dev/null
timeout 300 python bench.py --inplace --no-e2e --no-cpu-baseline > gpurun_out/final/fwht_inplace.json 2>/dev/null
