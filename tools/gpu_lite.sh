set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 900 python -m pytest tests/test_gpu_apply.py tests/test_gpu_compression.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -3
: > gpurun_out/lite.txt
for r in 1; do for c in cfg0 cfg1_unitxi cfg1 cfg3; do for f in 63 1087 65599; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --flags $f 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', $f, round(d['ms_per_step']*1e3,2))" >> gpurun_out/lite.txt
done; done; done
cat gpurun_out/lite.txt
