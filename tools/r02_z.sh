# whole-region single-n rates of the fused quantization (the sweep's per-n breakdown comes from
# back-to-back launches after the timed region and reads lower)
O=gpurun_out/r02_z
mkdir -p $O
for q in int4 e4m3 int8; do for n in 128 256 512 1024 2048 4096 8192 16384 32768; do
  timeout 120 python bench.py --workload quant-$q --ns $n --no-e2e --no-cpu-baseline --steps 30 > $O/x.json 2>/dev/null
  python -c "
import json
d=json.loads(open('$O/x.json').read().strip().splitlines()[-1]); print('$q', $n, d['value'], (d.get('clocks') or {}).get('sm_mhz'))
" | tee -a $O/single_n.txt
done; done
