# packed 16-bit phase-B storage (HC_QPACK_N) with more CTAs per SM, fused quantization A/B
build() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared -I include $1 -o paper_2412_08832_b200/libhadacore.so paper_2412_08832_b200/csrc/hadacore.cu 2>/dev/null; }
for v in "" "-DHC_QPACK_N=16384 -DHC_QTUNE -DHC_QTUNE_N=16384 -DHC_QNT=8 -DHC_QTKB=32 -DHC_QST=2 -DHC_QCTAS=3" "-DHC_QPACK_N=32768" "-DHC_QPACK_N=8192 -DHC_QTUNE -DHC_QTUNE_N=8192 -DHC_QNT=8 -DHC_QTKB=32 -DHC_QST=2 -DHC_QCTAS=3" ""; do
  build "$v"
  for q in e4m3 int8; do
    timeout 300 python bench.py --workload quant-$q --ns 8192,16384,32768 --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/ab.json 2>/dev/null
    python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('${v:-default}', '$q', d['per_n_GBps']['fp16'], d['per_n_GBps']['bf16'])
"
  done
done
