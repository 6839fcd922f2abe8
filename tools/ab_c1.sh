# C1 latency vs tile size (HC_TUNE: nt, tile KiB, stages for every n; only n = 256 is launched)
build() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared -I include $1 -o paper_2412_08832_b200/libhadacore.so paper_2412_08832_b200/csrc/hadacore.cu 2>/dev/null; }
for v in "" "-DHC_TUNE -DHC_NT=8 -DHC_TILE_KB=4 -DHC_STAGES=2 -DHC_U=1 -DHC_CTAS=1" "-DHC_TUNE -DHC_NT=8 -DHC_TILE_KB=8 -DHC_STAGES=2 -DHC_U=1 -DHC_CTAS=1" "-DHC_TUNE -DHC_NT=4 -DHC_TILE_KB=2 -DHC_STAGES=2 -DHC_U=1 -DHC_CTAS=1" ""; do
  build "$v"
  python bench.py --workload c1 > gpurun_out/c1.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/c1.json').read()); print('$v' or 'default', d['value'], 'us warm', d['cold_us'], 'us cold')
"
done
