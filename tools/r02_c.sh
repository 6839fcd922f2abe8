# round 2 (c): new edge/torch-op tests; mid-size sweep of the QT_MIDM variants; bank-conflict
# attribution (TMA store removed: HC_STG_OUT build) -- the library swap is the LAST step
set -x
O=gpurun_out/r02_c
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_gpu_torch_ops.py -q > $O/pytest_new.txt 2>&1; echo "rc=$?" >> $O/pytest_new.txt
L=$(ls build/mid/*.so | tr '\n' ',' | sed 's/,$//')
timeout 1200 python tools/midsize.py --libs $L --ns 256,512,1024,2048,4096,8192,16384,32768 --ks 22,23,24,25,26 --repeats 3 --out $O/midsize.json > $O/midsize.txt 2>&1
M="l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__sass_inst_executed_op_shared_ld.sum,smsp__sass_inst_executed_op_shared_st.sum,memory_l1_wavefronts_shared,memory_l1_wavefronts_shared_ideal,gpu__time_duration.sum"
timeout 600 ncu --metrics $M --clock-control none -k regex:fwht -s 4 -c 4 --csv python tools/ncu_one.py 256,1024 f16,bf16 > $O/conf_default.csv 2>&1
cp build/diag/stgout.so paper_2412_08832_b200/libhadacore.so
timeout 600 ncu --metrics $M --clock-control none -k regex:fwht -s 4 -c 4 --csv python tools/ncu_one.py 256,1024 f16,bf16 > $O/conf_stgout.csv 2>&1
