# Round-2 (second session) evidence refresh: GPU suite, smoke, bench lines for
# every config, DRAM traffic for the K2 config, launch list, full captures of
# k2_flow (Gauss tiles) and k5_id, factorization phase timings.
set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
make -q -C paper_1908_09376_b200 checked || make -C paper_1908_09376_b200 -j16 checked >/dev/null || exit 9
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rA > gpurun_out/r2c_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2c_tests.log
grep -E "passed|failed" gpurun_out/r2c_tests.log | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2c_smoke.log; tail -2 gpurun_out/r2c_smoke.log
: > gpurun_out/r2c_bench.jsonl
for c in cfg1 cfg0 cfg2 cfg3 cfg4 cfg1_unitxi; do timeout 600 python bench.py --config $c >> gpurun_out/r2c_bench.jsonl 2>gpurun_out/r2c_bench_$c.err; echo "bench $c rc=$?"; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in cfg4; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:'k1_flow|k2_flow|k1_coop' -s 4 -c 2 --csv --log-file gpurun_out/r2c_traffic_$c.csv python bench.py --config $c --steps 2 --warmup 4 --no-cpu-baseline --no-accuracy > gpurun_out/r2c_traffic_$c.log 2>&1; echo "ncu $c rc=$?"
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r2c_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/r2c_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k2_flow -s 2 -c 1 -f -o gpurun_out/r2c_k2_flow python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/r2c_k2.log 2>&1; echo "k2 full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k5_id -s 1 -c 1 -f -o gpurun_out/r2c_k5 python tools/k3_bench.py cfg1 > gpurun_out/r2c_k5.log 2>&1; echo "k5 full rc=$?"
MIDBF_FACT_TIMING=1 MIDBF_ID_TIMING=1 timeout 900 python tools/fact_timing.py cfg1 cfg3 > gpurun_out/r2c_fact.txt 2>&1; echo "fact rc=$?"
