# evict-first store hint A/B on the metric's sweep (paired: variants alternate)
build() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared -I include $1 -o paper_2412_08832_b200/libhadacore.so paper_2412_08832_b200/csrc/hadacore.cu 2>/dev/null; }
for rep in 1 2 3; do
for v in "-DHC_STORE_HINT=0" "-DHC_STORE_HINT=1"; do
  build "$v"
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$rep', '$v', d['value'], d['per_n_GBps']['fp16'])
"
done
done
