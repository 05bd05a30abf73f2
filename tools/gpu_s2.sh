set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 900 python -m pytest tests/test_gpu_ids.py tests/test_gpu_fullsize.py tests/test_gpu_lowrank.py tests/test_gpu_sample.py -q -x -p no:cacheprovider > gpurun_out/s18_tests.txt 2>&1; tail -2 gpurun_out/s18_tests.txt
timeout 600 python tools/fact_timing.py cfg1 cfg1_unitxi cfg3 > gpurun_out/s18_fact.txt 2>&1
