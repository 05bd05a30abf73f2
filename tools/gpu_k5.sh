# K5 change check: ID / factorization parity tests, then the factorize figures of the bench lines
set -o pipefail; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider -k "${K5_TESTS:-ids or fullsize or checked or sample or lowrank or golden}" > gpurun_out/k5_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/k5_tests.log
: > gpurun_out/k5_bench.jsonl
for c in ${K5_CFGS:-cfg1 cfg3 cfg1_unitxi cfg2}; do timeout 600 python bench.py --config $c --no-cpu-baseline >> gpurun_out/k5_bench.jsonl 2>gpurun_out/k5_bench_$c.err; echo "bench $c rc=$?"; done
python - <<'P'
import json
for l in open('gpurun_out/k5_bench.jsonl'):
    if not l.startswith('{'): continue
    d=json.loads(l); f=d['factorize']; k=f['k3_sampling']
    print(d['config']['workload'], 'factorize', f['seconds'], 'lib', f['library_seconds'], 'k5', k['k5_device_seconds'], 'ids gpu/host', f['ids_on_gpu'], f['ids_on_host'], 'acc', d.get('accuracy',{}).get('eps_b_device_sampled'), d.get('accuracy',{}).get('eps_b_host_sampled'))
P
