set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 600 python bench.py > gpurun_out/r1b_cfg1.json 2> gpurun_out/r1b_cfg1.err || { tail -5 gpurun_out/r1b_cfg1.err; exit 1; }
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1b_plain.json 2>&1 || exit 2
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1_launches.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k1_flow -s 5 -c 1 -f -o gpurun_out/r1_k1_flow python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1_k1_ncu.log 2>&1
ls -la gpurun_out/r1_k1_flow.ncu-rep gpurun_out/r1_launches.csv; cat gpurun_out/r1b_cfg1.json | head -c 600
