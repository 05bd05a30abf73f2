set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
B=131135
timeout 300 python tools/flow_ab.py cfg1_unitxi $B $((B+65536)) $((B+65536-48+16)) --rounds 7 > gpurun_out/s17_ab.txt 2>&1
timeout 300 python tools/flow_ab.py cfg1_unitxi $B $((B+65536)) --transpose --rounds 5 >> gpurun_out/s17_ab.txt 2>&1
timeout 300 python tools/flow_ab.py cfg0 $B $((B+524288)) $((B+524288+65536)) --rounds 7 >> gpurun_out/s17_ab.txt 2>&1
