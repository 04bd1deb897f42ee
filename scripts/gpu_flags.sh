cd $GRAFT_REPO_ROOT
for f in 0 4 2 6; do
echo "== flags $f"
for cfg in c4 c3; do KAN_DBG_FLAGS=$f timeout -s KILL 60 python scripts/prof_layer.py --config $cfg --iters 5 2>&1 | tail -3 | tr '\n' ' '; echo; done
done
