set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 900 python -m pytest tests/test_gpu_ids.py tests/test_gpu_sample.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -2
: > gpurun_out/k5exp.txt
for v in 4,0 4,2 4,3 8,0 8,1; do
  MIDBF_K5=$v timeout 300 python tools/k3_bench.py cfg1 cfg3 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    if d.get('kernel')=='k3': print('$v', d['workload'], 'k5 ms %.2f'%(1e3*d['k5_seconds']), 'k3 ms %.3f'%(1e3*d['k3_seconds']), 'fac s %.3f'%d['factorize_seconds'], d['ids_on_gpu'], d['ids_on_host'])
    else: print('$v', d['workload'], 'k4 %.3g entries/s'%d['entries_per_s'])
" >> gpurun_out/k5exp.txt
done
cat gpurun_out/k5exp.txt
