# ncu --set full of one C3 step (18 launches) on the final build -> profiles summary + roofline.traffic JSON
set -x
O=gpurun_out/r02_ncu_c3
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fwht -s 18 -c 18 -o $O/c3 \
  python tools/ncu_one.py > $O/ncu.log 2>&1
tail -2 $O/ncu.log
