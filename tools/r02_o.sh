# round 2 (o): full GPU suite + smoke + bench lines on the routed build (tcgen05 quant for n >= 16384)
set -x
O=gpurun_out/r02_o
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
timeout 400 python bench.py > $O/fwht.json 2> $O/fwht.err
for q in e4m3 int8 int4; do
  timeout 300 python bench.py --workload quant-$q --no-e2e --no-cpu-baseline > $O/quant-$q.json 2> $O/quant-$q.err
done
