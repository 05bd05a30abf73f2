# Round-2 check: GPU suite, smoke, cfg1 bench, compute-sanitizer (memcheck, synccheck, racecheck) on small cases.
set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r2a_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2a_tests.log
tail -15 gpurun_out/r2a_tests.log
timeout 300 python bench.py --config cfg1 > gpurun_out/r2a_bench.jsonl 2>gpurun_out/r2a_bench.err; echo "bench rc=$?"
cat gpurun_out/r2a_bench.jsonl | cut -c1-400
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > gpurun_out/r2a_sanitize_$tool.log 2>&1; echo "$tool rc=$?"
  tail -4 gpurun_out/r2a_sanitize_$tool.log
done
