# Round-2 refresh (second session, final: K2 tiles, wait hint, stage table in smem): GPU suite, smoke, bench lines for
# every config, the reference arm at cfg1, launch list, factorization phases.
set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
make -q -C paper_1908_09376_b200 checked || make -C paper_1908_09376_b200 -j16 checked >/dev/null || exit 9
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rA > gpurun_out/r2f_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2f_tests.log
grep -E "passed|failed" gpurun_out/r2f_tests.log | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2f_smoke.log; tail -2 gpurun_out/r2f_smoke.log
: > gpurun_out/r2f_bench.jsonl
for c in cfg1 cfg0 cfg2 cfg3 cfg4 cfg1_unitxi; do timeout 600 python bench.py --config $c >> gpurun_out/r2f_bench.jsonl 2>gpurun_out/r2f_bench_$c.err; echo "bench $c rc=$?"; done
timeout 900 python bench.py --impl reference --config cfg1 --steps 20 --warmup 3 > gpurun_out/r2f_ref_cfg1.jsonl 2>gpurun_out/r2f_ref_cfg1.err; echo "ref cfg1 rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/r2f_launches.log 2>&1; echo "launches rc=$?"
MIDBF_FACT_TIMING=1 MIDBF_ID_TIMING=1 timeout 900 python tools/fact_timing.py cfg1 > gpurun_out/r2f_fact.txt 2>&1; echo "fact rc=$?"
