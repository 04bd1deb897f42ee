cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests -m gpu -q -x --timeout 60 --timeout-method=thread -p no:cacheprovider > /tmp/tall.log 2>&1; echo PYTEST $?; tail -3 /tmp/tall.log | cut -c1-300
for cfg in c4 c2 c1 c3 c3bf16; do echo "== $cfg"; timeout -s KILL 60 python scripts/prof_layer.py --config $cfg --iters 10 2>&1 | tail -3 | tr '\n' ' '; echo; done
echo "== c5"; timeout -s KILL 120 python scripts/prof_layer.py --config c5 --iters 3 2>&1 | tail -21 | awk '{print $3}' | tr '\n' ' '
