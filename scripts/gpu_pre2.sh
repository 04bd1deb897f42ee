cd $GRAFT_REPO_ROOT
for M in 67108864 999999999999; do
KAN_LEVEL_PREPASS_MIN=$M timeout -s KILL 300 python bench.py --config c3 --steps 100 --warmup 5 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err
python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('$M', round(d['value']),round(d['ms_per_step']*1e3,1),'us',round(r['frac'],3),[round(v*1e3,1) for v in r['layer_avg_ms']], d['gpu_launches']/d['steps'])"
done
