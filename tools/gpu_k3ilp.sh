set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 900 python -m pytest tests/test_gpu_sample.py tests/test_gpu_ids.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/k3_bench.py cfg1 cfg2 cfg3 2>&1 | cut -c1-300
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,launch__grid_size,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:'k3_|k4_direct|k5_id' --csv --log-file gpurun_out/k3_counters.csv python tools/k3_bench.py cfg1 cfg2 cfg3 > gpurun_out/k3_counters.log 2>&1; echo "ncu counters rc=$?"
