# A/B of prebuilt libraries, interleaved: bash tools/ab_so.sh "<bench args>" a.so b.so ...  (ROUNDS=2)
args=$1; shift
for r in $(seq ${ROUNDS:-2}); do
  for so in "$@"; do
    cp "$so" paper_2412_08832_b200/libhadacore.so
    timeout 300 python bench.py $args --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/ab.json 2>/dev/null
    python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$so', '$args', d['value'], d.get('per_n_GBps'))
"
  done
done
