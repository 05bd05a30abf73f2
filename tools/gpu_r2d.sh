set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 300 python -m pytest tests/test_gpu_apply.py -m gpu -q -x -p no:cacheprovider -k "two_plans" > gpurun_out/r2d_t1.log 2>&1; echo "two-plan rc=$?"; tail -2 gpurun_out/r2d_t1.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2d_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2d_tests.log
for c in cfg1 cfg0; do timeout 300 python tools/flow_ab.py $c 131135 63 --rounds 11 --reps 20 2>&1 | tail -2; done
timeout 300 python bench.py --config cfg1 --no-accuracy > gpurun_out/r2d_bench.jsonl 2>gpurun_out/r2d_bench.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/r2d_bench.jsonl
