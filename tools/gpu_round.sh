# One refresh pass: all GPU tests, smoke, every bench config, the reference
# arm, K3/K4 counters, launch list + k1_flow / k3 ncu captures.
set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/full_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/full_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/full_smoke.log
tail -3 gpurun_out/full_tests.log; tail -2 gpurun_out/full_smoke.log
: > gpurun_out/full_bench.jsonl
for c in cfg1 cfg0 cfg2 cfg3 cfg4 cfg1_unitxi; do timeout 400 python bench.py --config $c >> gpurun_out/full_bench.jsonl 2>gpurun_out/full_bench_$c.err; echo "$c rc=$?"; done
timeout 300 python bench.py --impl reference >> gpurun_out/full_bench.jsonl 2>gpurun_out/full_bench_ref.err
wc -l gpurun_out/full_bench.jsonl
if [ -n "$PROF" ]; then
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,launch__grid_size,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:'k3_|k4_direct' --csv --log-file gpurun_out/k3_counters.csv python tools/k3_bench.py cfg1 cfg2 cfg3 > gpurun_out/k3_counters.log 2>&1; echo "ncu counters rc=$?"
timeout 600 python tools/k3_bench.py cfg1 cfg2 cfg3 > gpurun_out/k3_bench.jsonl 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k3_sample_ws_s' -s 2 -c 1 -f -o gpurun_out/r1_k3 python tools/k3_bench.py cfg1 > gpurun_out/k3_full.log 2>&1; echo "ncu k3 rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1_launches.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k1_flow -s 5 -c 1 -f -o gpurun_out/r1_k1_flow python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1_k1_ncu.log 2>&1; echo "k1 ncu rc=$?"
fi
if [ -n "$PROF" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k4_direct_s' -c 1 -f -o gpurun_out/r1_k4 python tools/k3_bench.py cfg1 > gpurun_out/k4_full.log 2>&1; echo "ncu k4 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k5_id' -s 1 -c 1 -f -o gpurun_out/r1_k5 python tools/k3_bench.py cfg1 > gpurun_out/k5_full.log 2>&1; echo "ncu k5 rc=$?"
fi
