# Round-2 final refresh: GPU suite, smoke, every bench config, the reference
# arm for every config, ncu DRAM traffic per config, launch list, full captures.
set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
make -q -C paper_1908_09376_b200 checked || make -C paper_1908_09376_b200 -j16 checked >/dev/null || exit 9
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rA > gpurun_out/r2z_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2z_tests.log
grep -E "passed|failed|eps_b" gpurun_out/r2z_tests.log | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2z_smoke.log; tail -2 gpurun_out/r2z_smoke.log
: > gpurun_out/r2z_bench.jsonl
for c in cfg1 cfg0 cfg2 cfg3 cfg4 cfg1_unitxi; do timeout 600 python bench.py --config $c >> gpurun_out/r2z_bench.jsonl 2>gpurun_out/r2z_bench_$c.err; echo "bench $c rc=$?"; done
: > gpurun_out/r2z_ref.jsonl
for c in cfg1 cfg0 cfg2 cfg3 cfg4 cfg1_unitxi; do timeout 900 python bench.py --impl reference --config $c --steps 20 --warmup 3 >> gpurun_out/r2z_ref.jsonl 2>gpurun_out/r2z_ref_$c.err; echo "ref $c rc=$?"; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in cfg1 cfg0 cfg2 cfg3 cfg4 cfg1_unitxi; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:'k1_flow|k2_flow|k1_coop' -s 4 -c 2 --csv --log-file gpurun_out/r2z_traffic_$c.csv python bench.py --config $c --steps 2 --warmup 4 --no-cpu-baseline --no-accuracy > gpurun_out/r2z_traffic_$c.log 2>&1; echo "ncu $c rc=$?"
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r2z_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/r2z_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1_flow -s 6 -c 1 -f -o gpurun_out/r2z_k1_flow python bench.py --steps 2 --warmup 4 --no-cpu-baseline --no-accuracy > gpurun_out/r2z_k1.log 2>&1; echo "k1 full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1_coop -s 6 -c 1 -f -o gpurun_out/r2z_k1_coop python bench.py --config cfg0 --steps 2 --warmup 4 --no-cpu-baseline --no-accuracy > gpurun_out/r2z_coop.log 2>&1; echo "coop full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k2_flow -s 2 -c 1 -f -o gpurun_out/r2z_k2_flow python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/r2z_k2.log 2>&1; echo "k2 full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k5_id -s 1 -c 1 -f -o gpurun_out/r2z_k5 python tools/k3_bench.py cfg1 > gpurun_out/r2z_k5.log 2>&1; echo "k5 full rc=$?"
