cd $GRAFT_REPO_ROOT
for f in 0 8 2 10; do echo "== flags $f"; KAN_LEVEL_PREPASS_MIN=999999999999 KAN_DBG_FLAGS=$f timeout -s KILL 120 python scripts/prof_layer.py --config c3 --iters 3 2>&1 | tail -3 | tr '\n' ' '; echo; done
