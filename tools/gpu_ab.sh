set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 900 python -m pytest tests/test_gpu_apply.py tests/test_golden.py -q -x --timeout 600 -p no:cacheprovider -k "identity or golden" > gpurun_out/ab_tests0.log 2>&1; echo "tests0 rc=$?" >> gpurun_out/ab_tests0.log
tail -3 gpurun_out/ab_tests0.log
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
tail -3 gpurun_out/ab_tests.log
: > gpurun_out/ab_bench.jsonl
for fl in 63 575; do timeout 600 python bench.py --config cfg1 --flags $fl >> gpurun_out/ab_bench.jsonl 2>gpurun_out/ab_$fl.err || tail -5 gpurun_out/ab_$fl.err; done
for c in cfg2 cfg3 cfg1_unitxi cfg0; do timeout 600 python bench.py --config $c --no-cpu-baseline >> gpurun_out/ab_bench.jsonl 2>gpurun_out/ab_$c.err || tail -5 gpurun_out/ab_$c.err; done
python - <<'PY'
import json
for l in open('gpurun_out/ab_bench.jsonl'):
    d=json.loads(l); r=d['roofline']
    print(d['config']['workload'], round(d['value']), 'us', round(d['ms_per_step']*1e3,1), 'frac', round(r['frac'],3), 'fact_eq', round(r.get('factor_equivalent_gbs',0)), 'flowMB', round(sum(s['flow_mb'] for s in d['stages']),1), [round(s['flow_mb'],1) for s in d['stages']], 'err', d.get('rel_l2_vs_ref'))
PY
