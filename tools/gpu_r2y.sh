# After the K5 changes: GPU suite, smoke, the default bench line, launch list, K5 full capture
set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
make -q -C paper_1908_09376_b200 checked || make -C paper_1908_09376_b200 -j16 checked >/dev/null || exit 9
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rA > gpurun_out/r2y_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2y_tests.log
grep -E "passed|failed|eps_b" gpurun_out/r2y_tests.log | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2y_smoke.log; tail -2 gpurun_out/r2y_smoke.log
: > gpurun_out/r2y_bench.jsonl
for c in cfg1 cfg3 cfg2 cfg1_unitxi; do timeout 600 python bench.py --config $c >> gpurun_out/r2y_bench.jsonl 2>gpurun_out/r2y_bench_$c.err; echo "bench $c rc=$?"; done
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r2y_ref.jsonl 2>gpurun_out/r2y_ref.err; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r2y_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/r2y_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k5_id -s 1 -c 1 -f -o gpurun_out/r2y_k5 python tools/k3_bench.py cfg1 > gpurun_out/r2y_k5.log 2>&1; echo "k5 full rc=$?"
