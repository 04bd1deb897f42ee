cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python -m pytest tests/test_gpu_conv.py -m gpu -q --timeout 120 --timeout-method=thread -p no:cacheprovider > /tmp/tc.log 2>&1; echo PYTEST_CONV $?; grep -E "^E |FAILED|passed|failed" /tmp/tc.log | head -8
run() { timeout -s KILL 120 python scripts/prof_layer.py --config c5 --iters 3 > /tmp/p5.log 2>&1; tail -21 /tmp/p5.log | awk -v s="$1" '{t+=$3; printf "%s ", $3} END {print " <-", s, "total", t}'; }
run base
KAN_DBG_FLAGS=60 run mma_only
KAN_DBG_FLAGS=62 run skeleton
KAN_DBG_FLAGS=2 run nomma
timeout -s KILL 120 python scripts/prof_layer.py --config c4 --iters 20 | tail -1
