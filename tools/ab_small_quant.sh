# small-n (n = 2..64) fused-quantization launch table A/B:
#   QS="e4m3 int4" bash tools/ab_small_quant.sh default 64:16,32,4,1 0:8,16,3,2 ...   (n = 0: every n)
build() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared -I include $1 -o paper_2412_08832_b200/libhadacore.so paper_2412_08832_b200/csrc/hadacore.cu 2>/dev/null || echo "BUILD FAILED $1"; }
run() { timeout 300 python bench.py --workload quant-$2 --ns ${NS:-2,4,8,16,32,64} --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$1', '$2', d['value'], d['per_n_GBps']['fp16'], d['per_n_GBps']['bf16'])
"; }
for v in "${@}"; do
  if [ "$v" = "default" ]; then build ""; else qn=${v%%:*}; IFS=, read nt tkb st uu <<< "${v#*:}"; build "-DHC_SQTUNE -DHC_SQTUNE_N=$qn -DHC_SQNT=$nt -DHC_SQTKB=$tkb -DHC_SQST=$st -DHC_SQU=$uu"; fi
  for q in ${QS:-e4m3 int4}; do run "$v" $q; done
done
build ""
