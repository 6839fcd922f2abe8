# fp32 n = 2^15 cluster kernel: consumer warps x groups A/B (tools/f32_pair_probe.py)
build() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared -I include $1 -o paper_2412_08832_b200/libhadacore.so paper_2412_08832_b200/csrc/hadacore.cu 2>/dev/null; }
for v in "-DHC_PAIR_NT=16 -DHC_PAIR_G=2" "-DHC_PAIR_NT=12 -DHC_PAIR_G=3" "-DHC_PAIR_NT=8 -DHC_PAIR_G=2" "-DHC_PAIR_NT=16 -DHC_PAIR_G=2"; do
  build "$v"; echo "$v"; python tools/f32_pair_probe.py | head -1
done
