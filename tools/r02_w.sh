O=gpurun_out/r02_w
mkdir -p $O
for q in int4 e4m3; do for n in 4096 8192; do
  for so in build/tcab/cur.so build/tcab/min4096.so; do
    cp $so paper_2412_08832_b200/libhadacore.so
    timeout 120 python bench.py --workload quant-$q --ns $n --no-e2e --no-cpu-baseline --steps 30 > $O/x.json 2>/dev/null
    python -c "
import json
d=json.loads(open('$O/x.json').read().strip().splitlines()[-1]); print('$q', $n, '$so', d['value'])
" | tee -a $O/pern.txt
  done
done; done
cp build/tcab/cur.so paper_2412_08832_b200/libhadacore.so
