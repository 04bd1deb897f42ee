cd $GRAFT_REPO_ROOT
for sl in 8 16 32 64; do for c in c1st c2st; do KAN_ST_SLICES=$sl timeout -s KILL 300 python bench.py --config $c --steps 3000 --warmup 30 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('slices $sl $c', round(d['ms_per_step']*1e3,2), 'us')"; done; done
for sl in 1 2 4 8; do KAN_ST_SLICES=$sl timeout -s KILL 300 python bench.py --config c4st --steps 300 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('slices $sl c4st', round(d['ms_per_step']*1e3,2), 'us')"; done
