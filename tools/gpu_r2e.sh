set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 900 python -m pytest tests/test_gpu_stress.py tests/test_gpu_apply.py -m gpu -q -x -p no:cacheprovider -k "${TESTK:-}" > gpurun_out/r2e_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r2e_tests.log
for c in ${CONFIGS:-cfg0 cfg1_unitxi cfg1 cfg3}; do timeout 300 python tools/flow_ab.py $c 131135 393279 --rounds 9 --reps 20 2>&1 | grep -E "median|diff"; done
