# Round-2 refresh: GPU suite, smoke, every bench config (with accuracy), the
# reference arm for every config, ncu DRAM traffic of the dominant kernel per config.
set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rA -k "${TESTK:-}" > gpurun_out/r2b_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2b_tests.log
grep -E "passed|failed|eps_b" gpurun_out/r2b_tests.log | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2b_smoke.log; tail -2 gpurun_out/r2b_smoke.log
: > gpurun_out/r2b_bench.jsonl
for c in ${CONFIGS:-cfg1 cfg0 cfg2 cfg3 cfg4 cfg1_unitxi}; do timeout 600 python bench.py --config $c >> gpurun_out/r2b_bench.jsonl 2>gpurun_out/r2b_bench_$c.err; echo "bench $c rc=$?"; done
: > gpurun_out/r2b_ref.jsonl
for c in ${CONFIGS:-cfg1 cfg0 cfg2 cfg3 cfg4 cfg1_unitxi}; do timeout 900 python bench.py --impl reference --config $c --steps 20 --warmup 3 >> gpurun_out/r2b_ref.jsonl 2>gpurun_out/r2b_ref_$c.err; echo "ref $c rc=$?"; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in ${CONFIGS:-cfg1 cfg0 cfg2 cfg3 cfg4 cfg1_unitxi}; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:'k1_flow|k2_flow' -s 4 -c 2 --csv --log-file gpurun_out/r2b_traffic_$c.csv python bench.py --config $c --steps 2 --warmup 4 --no-cpu-baseline --no-accuracy > gpurun_out/r2b_traffic_$c.log 2>&1; echo "ncu $c rc=$?"
done
