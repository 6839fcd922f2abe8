# transform launch-table A/B for one n: bash tools/ab_transform_tune.sh default 16384:16,32,6,1 ...
build() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared -I include $1 -o paper_2412_08832_b200/libhadacore.so paper_2412_08832_b200/csrc/hadacore.cu 2>/dev/null; }
for v in "${@}"; do
  if [ "$v" = "default" ]; then build ""; else tn=${v%%:*}; IFS=, read nt tkb st ct <<< "${v#*:}"; build "-DHC_TTUNE -DHC_TTUNE_N=$tn -DHC_TNT=$nt -DHC_TTKB=$tkb -DHC_TST=$st -DHC_TCTAS=$ct"; fi
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['per_n_GBps']['fp16']['16384'], d['per_n_GBps']['bf16']['16384'], d['per_n_GBps']['fp16']['32768'], d['per_n_GBps']['bf16']['32768'])
"
done
