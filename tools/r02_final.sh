# round 2 final evidence on the committed build: full GPU suite, smoke, every bench.py workload
# (JSON lines for profiles/r02_final), ncu launch list of the default bench, 2-rank torchrun checks
set -x
O=gpurun_out/r02_final
mkdir -p $O
timeout 60 python tools/pp_probe.py > $O/quick.txt 2>&1; echo "quick rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
tail -2 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 400 python bench.py > $O/fwht.json 2> $O/fwht.err
for w in quant-e4m3 quant-int8 quant-int4 f32 small c1 c2 c4 c5 qk-rotate qk-quant lab; do
  timeout 400 python bench.py --workload $w --no-e2e --no-cpu-baseline > $O/$w.json 2> $O/$w.err
done
for q in e4m3 int8 int4; do
  timeout 300 python bench.py --workload quant-$q --ns 2,4,8,16,32,64 --no-e2e --no-cpu-baseline > $O/quant-$q-small.json 2>/dev/null
done
timeout 300 python bench.py --inplace --no-e2e --no-cpu-baseline > $O/fwht_inplace.json 2>/dev/null
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > $O/reference.json 2> $O/reference.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e > $O/torchrun2_fwht.json 2> $O/torchrun2_fwht.err; echo "rc=$?" >> $O/torchrun2_fwht.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 \
  bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e --misshard > $O/torchrun2_misshard.json 2> $O/torchrun2_misshard.err; echo "rc=$?" >> $O/torchrun2_misshard.err
