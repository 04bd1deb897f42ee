cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -q -x --timeout 60 --timeout-method=thread -p no:cacheprovider > gpurun_out/tall.log 2>&1; echo PYTEST $?
tail -4 gpurun_out/tall.log
for cfg in c4 c2 c3; do echo "== $cfg"; timeout -s KILL 60 python scripts/prof_layer.py --config $cfg --iters 10 2>&1 | tail -3; done
echo "== c5"; timeout -s KILL 120 python scripts/prof_layer.py --config c5 --iters 3 2>&1 | tail -21 | tr '\n' ' '
