# A/B of env variants: per-stage device times (tools/ab_stage.py) -> gpurun_out/ab.txt
mkdir -p gpurun_out
VAR=${VAR:-SVR_COMP_COOP}
for w in ${WL:-cfg2 cfg3 cfg4}; do
 for c in ${VALS:-1 0}; do env $VAR=$c timeout 300 python tools/ab_stage.py $w 30 >> gpurun_out/ab.txt 2>&1; done
done
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest $TESTS -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "rc $?" >> gpurun_out/pytest.log; fi
