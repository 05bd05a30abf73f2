# K3 / K4 FP64 evidence: kernel-event throughput (tools/k3_bench.py) and ncu
# SASS FP64 counters of the staged sampler / direct-sum kernels.
set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 900 python -m pytest tests/test_gpu_sample.py tests/test_gpu_fullsize.py tests/test_gpu_apply.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/k3p_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/k3p_tests.log; tail -2 gpurun_out/k3p_tests.log
timeout 300 python tools/k3_bench.py cfg1 cfg2 cfg3 > gpurun_out/k3_bench.jsonl 2> gpurun_out/k3_bench.err; echo "k3 rc=$?"; cat gpurun_out/k3_bench.jsonl
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_fp64_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:'k3_|k4_direct' --csv --log-file gpurun_out/k3_counters.csv python tools/k3_bench.py cfg1 cfg2 cfg3 > gpurun_out/k3_counters.log 2>&1; echo "ncu counters rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k3_sample_ws_s' -s 2 -c 1 -f -o gpurun_out/r1_k3 python tools/k3_bench.py cfg1 > gpurun_out/k3_full.log 2>&1; echo "ncu k3 full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k4_direct_s' -c 1 -f -o gpurun_out/r1_k4 python tools/k3_bench.py cfg1 > gpurun_out/k4_full.log 2>&1; echo "ncu k4 full rc=$?"
ls -la gpurun_out/*.ncu-rep
