set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
for c in cfg0 cfg1_unitxi cfg1; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-accuracy 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step']*1e3,2), d['host_issue_us_per_step'], d['e2e']['value'])"; done > gpurun_out/s29.txt
