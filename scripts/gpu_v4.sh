cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/t4.log 2>&1; echo PYTEST $?
tail -3 gpurun_out/t4.log
for cfg in c2 c1 c3 c3bf16; do echo "== $cfg"; timeout -s KILL 200 python scripts/prof_layer.py --config $cfg --iters 20; done
for f in 0 1 3; do echo "== flags $f"; KAN_DBG_FLAGS=$f timeout -s KILL 200 python scripts/timeline.py --config c3 --batch 16384 2>&1 | grep -i "layer 0" -A3 | head -4; KAN_DBG_FLAGS=$f timeout -s KILL 200 python scripts/timeline.py --config c2 --split 1 2>&1 | grep -i "layer 0" -A3 | head -4; done
