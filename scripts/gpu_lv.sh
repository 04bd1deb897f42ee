cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests -m gpu -q --timeout 120 --timeout-method=thread -p no:cacheprovider > /tmp/tall.log 2>&1; echo PYTEST $?; grep -E "^E |FAILED|passed|failed" /tmp/tall.log | head -6
for S in 1 0; do
KAN_LV_SIDECAR=$S timeout -s KILL 120 python scripts/prof_layer.py --config c5 --iters 3 > /tmp/p5.log 2>&1; tail -21 /tmp/p5.log | awk -v s=$S '{t+=$3; printf "%s ", $3} END {print " sidecar", s, "total", t}'
done
timeout -s KILL 300 python bench.py --config c3 --steps 100 --warmup 5 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err
python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('c3', round(d['value']),round(d['ms_per_step']*1e3,1),'us',round(r['frac'],3),[round(v*1e3,1) for v in r['layer_avg_ms']])"
