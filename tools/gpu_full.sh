set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/full_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/full_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/full_smoke.log
: > gpurun_out/full_bench.jsonl
for c in cfg1 cfg0 cfg2 cfg3 cfg4 cfg1_unitxi; do timeout 600 python bench.py --config $c >> gpurun_out/full_bench.jsonl 2>gpurun_out/full_bench_$c.err; done
timeout 300 python bench.py --impl reference >> gpurun_out/full_bench.jsonl 2>gpurun_out/full_bench_ref.err
if [ -n "$K2NCU" ]; then timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k2_flow -s 3 -c 1 -f -o gpurun_out/r1_k2_flow python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1_k2_ncu.log 2>&1; fi
tail -3 gpurun_out/full_tests.log; tail -2 gpurun_out/full_smoke.log; wc -l gpurun_out/full_bench.jsonl
