# A/B against an older build in tools/_build/old (git worktree): bench
# device times, alternating old / new, per config.
set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
: > gpurun_out/regress.txt
for r in 1 2; do for c in ${CONFIGS:-cfg2 cfg3 cfg1}; do
  for t in old new; do
    d=.; [ $t = old ] && d=tools/_build/old
    (cd $d && timeout 300 python bench.py --config $c --no-cpu-baseline --no-accuracy 2>/dev/null) | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', '$c', round(d['ms_per_step']*1e3,2), d['clocks']['sm_mhz'])" >> gpurun_out/regress.txt
  done
done; done
cat gpurun_out/regress.txt
[ -n "$FACT" ] && MIDBF_FACT_TIMING=1 MIDBF_ID_TIMING=1 timeout 600 python tools/fact_timing.py $FACT > gpurun_out/regress_fact.txt 2>&1
true
