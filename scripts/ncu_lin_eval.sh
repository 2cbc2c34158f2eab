cd /root/repo; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_linear -s 0 -c 2 -o gpurun_out/tc_dense4096 python scripts/ncu_linear.py 4096 > gpurun_out/ncu_lin.log 2>&1
tail -2 gpurun_out/ncu_lin.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:act_kernel -s 1 -c 1 -o gpurun_out/act_eval_b64 python scripts/ncu_target.py 64 > gpurun_out/ncu_ev.log 2>&1
tail -2 gpurun_out/ncu_ev.log
