cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests -m gpu -q -x --timeout 60 --timeout-method=thread -p no:cacheprovider > /tmp/tall.log 2>&1; echo PYTEST $?; tail -3 /tmp/tall.log | cut -c1-300
for cfg in c2 c1 c3; do echo "== $cfg"; timeout -s KILL 60 python scripts/prof_layer.py --config $cfg --iters 10 2>&1 | tail -3 | tr '\n' ' '; echo; done
