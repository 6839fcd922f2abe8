O=gpurun_out/r02_v
mkdir -p $O
timeout 60 python tools/pp_probe.py > $O/quick.txt 2>&1; echo "quick rc=$?"
timeout 400 python -m pytest tests/test_gpu_jitter.py tests/test_gpu_quant.py tests/test_gpu_edge.py -q -x > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt; tail -2 $O/pytest.txt
