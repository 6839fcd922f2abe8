# fused-quantization launch table A/B: bash tools/ab_quant_tune.sh default 0:8,16,3,3 16384:8,32,3,2 ...
build() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared -I include $1 -o paper_2412_08832_b200/libhadacore.so paper_2412_08832_b200/csrc/hadacore.cu 2>/dev/null; }
run() { timeout 300 python bench.py --workload quant-$1 --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$2', '$1', d['value'], d['per_n_GBps']['fp16'], d['per_n_GBps']['bf16'])
"; }
for v in "${@}"; do
  # v = "default" or "n:nt,tkb,st,ctas" (n = 0: every n in 512..8192)
  if [ "$v" = "default" ]; then build ""; else qn=${v%%:*}; IFS=, read nt tkb st ct uu <<< "${v#*:}"; build "-DHC_QTUNE -DHC_QTUNE_N=$qn -DHC_QNT=$nt -DHC_QTKB=$tkb -DHC_QST=$st -DHC_QCTAS=$ct -DHC_QU=${uu:-1}"; fi
  run e4m3 "$v"
done
