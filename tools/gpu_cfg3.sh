make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
mkdir -p gpurun_out; : > gpurun_out/cfg3.txt
for c in cfg3 cfg2 cfg1; do for f in 31 47 63; do
PYTHONFAULTHANDLER=1 timeout -s ABRT 90 python bench.py --config $c --no-cpu-baseline --steps 20 --flags $f > /tmp/o.json 2>/tmp/o.err; echo "$c flags=$f rc=$? $(python -c "import json; d=json.load(open('/tmp/o.json')); print(round(d['ms_per_step']*1e3,2), d['roofline']['frac'])" 2>/dev/null)" >> gpurun_out/cfg3.txt
done; done
timeout 600 python -m pytest tests/test_gpu_apply.py tests/test_gpu_compression.py -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -2 >> gpurun_out/cfg3.txt
cat gpurun_out/cfg3.txt
