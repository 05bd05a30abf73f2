# A/B of plan flag sets (tools/flow_ab.py) + the GPU suite
set -o pipefail; mkdir -p gpurun_out
make -q -C paper_1908_09376_b200 || make -C paper_1908_09376_b200 -j16 >/dev/null || exit 9
make -q -C paper_1908_09376_b200 checked || make -C paper_1908_09376_b200 -j16 checked >/dev/null || exit 9
OUT=gpurun_out/${AB_TAG:-ab}.txt; : > $OUT
while read -r c fl; do [ -z "$c" ] && continue; echo "== $c $fl" >> $OUT; timeout 600 python tools/flow_ab.py $c $fl --rounds ${AB_ROUNDS:-15} >> $OUT 2>&1; done <<< "$AB_CASES"
grep -v Warn $OUT
if [ -n "$AB_SUITE" ]; then timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/${AB_TAG:-ab}_suite.log 2>&1; echo "suite rc=$?"; tail -2 gpurun_out/${AB_TAG:-ab}_suite.log; fi
