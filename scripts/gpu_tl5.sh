cd $GRAFT_REPO_ROOT
for f in 2048; do echo "== c2 flags $f"; KAN_DBG_FLAGS=$f KAN_TIMELINE=1 timeout -s KILL 120 python scripts/timeline.py --config c2 2>&1 | grep -E "lastA|tmemfull|partials|reduced"; done
