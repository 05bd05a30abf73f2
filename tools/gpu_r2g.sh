# Round-2 third session: sanity of the restored tree (suite, smoke, cfg1 / cfg0 / unitxi bench lines)
set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
make -q -C paper_1908_09376_b200 checked || make -C paper_1908_09376_b200 -j16 checked >/dev/null || exit 9
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rA > gpurun_out/r2g_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2g_tests.log
grep -E "passed|failed" gpurun_out/r2g_tests.log | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2g_smoke.log
: > gpurun_out/r2g_bench.jsonl
for c in cfg1 cfg0 cfg1_unitxi; do timeout 600 python bench.py --config $c >> gpurun_out/r2g_bench.jsonl 2>gpurun_out/r2g_bench_$c.err; echo "bench $c rc=$?"; done
