# Session baseline: timelines and timing modes for cfg1 / cfg0 / cfg1_unitxi.
set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
for c in cfg1 cfg1_unitxi cfg0; do
  timeout 300 python tools/flow_timeline.py 131135 $c > gpurun_out/s1_tl_$c.txt 2>&1; echo "tl $c rc=$?"
  timeout 300 python tools/flow_ab.py $c 131135 131263 131327 131391 --rounds 7 > gpurun_out/s1_ab_$c.txt 2>&1; echo "ab $c rc=$?"
done
