cd $GRAFT_REPO_ROOT
for f in 0 2 8 10 16; do KAN_DBG_FLAGS=$f timeout -s KILL 300 python scripts/prof_layer.py --config c5 --iters 3 2>&1 | grep -E "layer (0|1|5):" | tr '\n' ' ' | sed "s/^/c5 flags $f: /"; echo; done
