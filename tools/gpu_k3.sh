set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 600 python -m pytest tests/test_gpu_sample.py tests/test_gpu_ids.py tests/test_gpu_lowrank.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/k3_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/k3_tests.log
tail -3 gpurun_out/k3_tests.log
PYTHONFAULTHANDLER=1 MIDBF_ID_TIMING=1 MIDBF_PLAN_TIMING=1 timeout -s ABRT 200 python bench.py --config cfg3 --no-cpu-baseline --steps 5 > gpurun_out/cfg3_dbg.json 2> gpurun_out/cfg3_dbg.err; echo "cfg3 rc=$?"
tail -c 300 gpurun_out/cfg3_dbg.json; tail -30 gpurun_out/cfg3_dbg.err | cut -c1-200
timeout 300 python tools/k3_bench.py cfg1 cfg2 > gpurun_out/k3_bench.jsonl 2> gpurun_out/k3_bench.err; echo "k3 rc=$?"
cat gpurun_out/k3_bench.jsonl
