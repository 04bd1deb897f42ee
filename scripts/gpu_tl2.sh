cd $GRAFT_REPO_ROOT
for s in 0 2 4 8; do echo "== c2 split $s"; KAN_TIMELINE=1 timeout -s KILL 120 python scripts/timeline.py --config c2 --split $s 2>&1 | tail -12; done
echo "== c1"; KAN_TIMELINE=1 timeout -s KILL 120 python scripts/timeline.py --config c1 2>&1 | tail -12
for s in 2 4 8; do timeout -s KILL 200 python bench.py --config c2 --steps 5000 --warmup 50 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('bench c2 default', round(d['ms_per_step']*1e3,2))"; break; done
