# n = 128 fused-quant config A/B on the contiguous (quant-e4m3) and strided (qk-quant) sweeps
build() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared -I include $1 -o paper_2412_08832_b200/libhadacore.so paper_2412_08832_b200/csrc/hadacore.cu 2>/dev/null; }
for v in "${@}"; do
  if [ "$v" = "default" ]; then build ""; else IFS=, read nt tkb st ct <<< "$v"; build "-DHC_QTUNE -DHC_QTUNE_N=128 -DHC_QNT=$nt -DHC_QTKB=$tkb -DHC_QST=$st -DHC_QCTAS=$ct"; fi
  for w in quant-e4m3 qk-quant; do
    timeout 300 python bench.py --workload $w --ns 128,256 --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/ab.json 2>/dev/null
    python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$v', '$w', d['per_n_GBps']['fp16']['128'], d['per_n_GBps']['bf16']['128'])
"
  done
done
