cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python -m pytest tests/test_gpu_conv.py -m gpu -q --timeout 120 --timeout-method=thread -p no:cacheprovider > /tmp/tc.log 2>&1; echo PYTEST_CONV $?; grep -E "^E |FAILED|passed|failed" /tmp/tc.log | head -8
for S in 2 1; do
KAN_CONV3_MC=$S timeout -s KILL 120 python scripts/prof_layer.py --config c5 --iters 3 > /tmp/p5.log 2>&1; tail -21 /tmp/p5.log | awk -v s=$S '{t+=$3; printf "%s ", $3} END {print " mc", s, "total", t}'
done
KAN_CONV3_MC=2 timeout -s KILL 120 python scripts/prof_layer.py --config c4 --iters 20 | tail -1
KAN_CONV3_MC=1 timeout -s KILL 120 python scripts/prof_layer.py --config c4 --iters 20 | tail -1
timeout -s KILL 600 python -m pytest tests -m gpu -q --timeout 120 --timeout-method=thread -p no:cacheprovider > /tmp/tall.log 2>&1; echo PYTEST $?; grep -E "^E |FAILED|passed|failed" /tmp/tall.log | head -6
