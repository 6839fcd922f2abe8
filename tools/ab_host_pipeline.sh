# host-buffer pipeline A/B: block size (MiB) x slots/streams
build() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared -I include $1 -o paper_2412_08832_b200/libhadacore.so paper_2412_08832_b200/csrc/hadacore.cu 2>/dev/null; }
for v in "16 4" "32 4" "8 8" "4 8" "64 2" "16 4"; do
  set -- $v
  build "-DHC_HOST_BLOCK_MB=$1 -DHC_HOST_SLOTS=$2"
  echo "block=$1MiB slots=$2"; python tools/pcie_probe.py | grep fwht_host
done
