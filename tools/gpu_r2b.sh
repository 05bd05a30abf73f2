# Round-2 (second session) refresh: GPU suite, smoke, bench lines for every
# config, ncu DRAM traffic per k1 config, launch list, full captures of the
# changed kernels (k1_flow at cfg1, k1_coop at cfg0, k5_id in a cfg1 factorization).
set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
make -q -C paper_1908_09376_b200 checked || make -C paper_1908_09376_b200 -j16 checked >/dev/null || exit 9
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rA > gpurun_out/r2b_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2b_tests.log
grep -E "passed|failed" gpurun_out/r2b_tests.log | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2b_smoke.log; tail -2 gpurun_out/r2b_smoke.log
: > gpurun_out/r2b_bench.jsonl
for c in cfg1 cfg0 cfg2 cfg3 cfg4 cfg1_unitxi; do timeout 600 python bench.py --config $c >> gpurun_out/r2b_bench.jsonl 2>gpurun_out/r2b_bench_$c.err; echo "bench $c rc=$?"; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in cfg1 cfg0 cfg2 cfg3 cfg1_unitxi; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:'k1_flow|k2_flow|k1_coop' -s 4 -c 2 --csv --log-file gpurun_out/r2b_traffic_$c.csv python bench.py --config $c --steps 2 --warmup 4 --no-cpu-baseline --no-accuracy > gpurun_out/r2b_traffic_$c.log 2>&1; echo "ncu $c rc=$?"
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r2b_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/r2b_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1_flow -s 6 -c 1 -f -o gpurun_out/r2b_k1_flow python bench.py --steps 2 --warmup 4 --no-cpu-baseline --no-accuracy > gpurun_out/r2b_k1.log 2>&1; echo "k1 full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k5_id -s 1 -c 1 -f -o gpurun_out/r2b_k5 python tools/k3_bench.py cfg1 > gpurun_out/r2b_k5.log 2>&1; echo "k5 full rc=$?"
