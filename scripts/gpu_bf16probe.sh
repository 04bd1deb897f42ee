cd $GRAFT_REPO_ROOT
for f in 0 4 6 7 8; do KAN_DBG_FLAGS=$f timeout -s KILL 300 python scripts/prof_layer.py --config c3bf16 --iters 3 2>&1 | tail -4 | head -1 | sed "s/^/bf16 flags $f: /"; done
for f in 0 4 6; do KAN_DBG_FLAGS=$f timeout -s KILL 300 python scripts/prof_layer.py --config c3 --iters 3 2>&1 | tail -4 | head -1 | sed "s/^/int8 flags $f: /"; done
