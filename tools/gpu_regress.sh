set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 900 python -m pytest tests/test_gpu_apply.py tests/test_gpu_compression.py tests/test_golden.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -2
: > gpurun_out/regress.txt
for r in 1 2; do for c in cfg0 cfg1_unitxi cfg1; do
  for t in old; do (cd tools/_build/$t && timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null) | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', '$c', round(d['ms_per_step']*1e3,2))" >> gpurun_out/regress.txt; done
  timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new', '$c', round(d['ms_per_step']*1e3,2))" >> gpurun_out/regress.txt
done; done
cat gpurun_out/regress.txt
