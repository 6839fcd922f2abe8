# round 2 (d): state of HEAD after the packed-FADD2 / mid-size commit: the full GPU suite, smoke,
# the default bench line, and the quant / f32 lines the next changes target
set -x
O=gpurun_out/r02_d
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 400 python bench.py > $O/fwht.json 2> $O/fwht.err
for q in e4m3 int8 int4; do
  timeout 300 python bench.py --workload quant-$q --no-e2e --no-cpu-baseline > $O/quant-$q.json 2> $O/quant-$q.err
done
timeout 300 python bench.py --workload f32 --no-e2e --no-cpu-baseline > $O/f32.json 2> $O/f32.err
