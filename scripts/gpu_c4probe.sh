cd $GRAFT_REPO_ROOT
for f in 0 62 58 26 16 2; do KAN_DBG_FLAGS=$f timeout -s KILL 300 python scripts/prof_layer.py --config c4 --iters 20 2>&1 | grep "layer 0" | sed "s/^/c4 flags $f: /"; done
