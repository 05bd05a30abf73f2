# PDL chain experiment: correctness (stress with chain) + interleaved A/B timing
set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
[ -n "$SKIPTEST" ] || timeout 900 python -m pytest tests/test_gpu_stress.py tests/test_gpu_apply.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2c_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2c_tests.log
for c in cfg1 cfg0 cfg1_unitxi cfg3 cfg2; do timeout 300 python tools/flow_ab.py $c 63 131135 --rounds 11 --reps 20 2>&1 | tail -3; done
