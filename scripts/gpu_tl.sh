cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests -m gpu -q -x --timeout 60 --timeout-method=thread -p no:cacheprovider > /tmp/tall.log 2>&1; echo PYTEST $?; tail -2 /tmp/tall.log
timeout -s KILL 60 python scripts/timeline.py --config c4 2>&1 | tail -12
timeout -s KILL 60 python scripts/timeline.py --config c2 2>&1 | tail -24
