set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
timeout 900 python tools/fact_timing.py cfg3 cfg1 cfg2 cfg0 > gpurun_out/s22_fact.txt 2>&1
