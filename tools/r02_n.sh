# per-(qtype, n) whole-region A/B: tcgen05 fused quantization vs the fwht_rows_kernel epilogue
O=gpurun_out/r02_n
mkdir -p $O
for q in e4m3 int8 int4; do for n in 4096 8192 16384 32768; do
  for so in build/tcdiag/old.so build/tcab/tc.so; do
    cp $so paper_2412_08832_b200/libhadacore.so
    timeout 120 python bench.py --workload quant-$q --ns $n --no-e2e --no-cpu-baseline --steps 30 > $O/x.json 2>/dev/null
    python -c "
import json
d=json.loads(open('$O/x.json').read().strip().splitlines()[-1]); print('$q', $n, '$so', d['value'])
" | tee -a $O/pern.txt
  done
done; done
cp build/tcab/tc.so paper_2412_08832_b200/libhadacore.so
