cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests -m gpu -q -x --timeout 60 --timeout-method=thread -p no:cacheprovider > /tmp/tall.log 2>&1; echo PYTEST $?; tail -1 /tmp/tall.log | cut -c1-300
for cfg in c2 c1; do
timeout -s KILL 300 python bench.py --config $cfg --steps 20000 --warmup 200 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err; echo "BENCH $cfg $?"
python -c "import json;d=json.load(open('/tmp/b.json'));print(d['value'],d['ms_per_step']*1e3,'us', d['gpu_launches']/d['steps'])"
done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/dur.csv python scripts/prof_layer.py --config c2 --iters 3 --nograph > /dev/null 2>&1; grep -o '"kan_[a-z_]*.*' /tmp/dur.csv | awk -F'","' '{print substr($1,1,30), $NF}' | tail -4
