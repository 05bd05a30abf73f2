set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2f_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
: > gpurun_out/r2f_bench.jsonl
for c in ${CONFIGS:-cfg1 cfg0 cfg1_unitxi}; do timeout 600 python bench.py --config $c >> gpurun_out/r2f_bench.jsonl 2>gpurun_out/r2f_bench_$c.err; echo "bench $c rc=$?"; done
