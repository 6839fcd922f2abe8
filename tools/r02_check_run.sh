# round 2: GPU tests + the new bench legs (c2, c4, c1 clocks, in-place check) + torchrun 2-rank
# self-check (gloo: both ranks share the one GPU) and its --misshard negative control
set -x
O=gpurun_out/r02_a
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python bench.py --steps 10 > $O/fwht.json 2> $O/fwht.err; echo "rc=$?" >> $O/fwht.err
for w in c2 c4 c1; do
  timeout 300 python bench.py --workload $w --steps 20 > $O/$w.json 2> $O/$w.err; echo "rc=$?" >> $O/$w.err
done
timeout 300 python bench.py --inplace --steps 5 --no-e2e --no-cpu-baseline > $O/fwht_inplace.json 2> $O/fwht_inplace.err
timeout 300 python bench.py --misshard --steps 2 --no-e2e --no-cpu-baseline > $O/misshard_n1.json 2> $O/misshard_n1.err; echo "rc=$?" >> $O/misshard_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e > $O/torchrun2_fwht.json 2> $O/torchrun2_fwht.err; echo "rc=$?" >> $O/torchrun2_fwht.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 \
  bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e --misshard > $O/torchrun2_misshard.json 2> $O/torchrun2_misshard.err; echo "rc=$?" >> $O/torchrun2_misshard.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --workload c5 --steps 2 --warmup 3 > $O/torchrun2_c5.json 2> $O/torchrun2_c5.err; echo "rc=$?" >> $O/torchrun2_c5.err
