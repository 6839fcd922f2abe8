# round 2 (q): jitter protocol tests, the new negative-control quant test, full GPU suite
set -x
O=gpurun_out/r02_q
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_jitter.py tests/test_gpu_edge.py -q -k "jitter or negative" > $O/pytest_jitter.txt 2>&1; echo "rc=$?" >> $O/pytest_jitter.txt
tail -5 $O/pytest_jitter.txt
