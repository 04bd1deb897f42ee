cd $GRAFT_REPO_ROOT
echo "== c2 flags16 (lastA := reduction loop done)"; KAN_DBG_FLAGS=16 KAN_TIMELINE=1 timeout -s KILL 120 python scripts/timeline.py --config c2 2>&1 | tail -11
echo "== c2 flags32 (tmemfull := cols staged)"; KAN_DBG_FLAGS=32 KAN_TIMELINE=1 timeout -s KILL 120 python scripts/timeline.py --config c2 2>&1 | tail -11
