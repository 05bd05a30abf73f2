set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
B=131135; P=16777216
for c in cfg0; do
  timeout 400 python tools/flow_ab.py $c $B $((B+P)) --rounds 15 > gpurun_out/s6_ab_$c.txt 2>&1; echo "ab $c rc=$?"
  timeout 400 python tools/flow_ab.py $c $B $((B+P)) --transpose --rounds 9 > gpurun_out/s6_abT_$c.txt 2>&1; echo "abT $c rc=$?"
done
timeout 600 python -m pytest tests/test_gpu_stress.py tests/test_gpu_apply.py -q -x -p no:cacheprovider 2>&1 | tail -2
