cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests -m gpu -q --timeout 120 --timeout-method=thread -p no:cacheprovider > /tmp/tall.log 2>&1; echo PYTEST $?; grep -E "^E |FAILED|passed|failed" /tmp/tall.log | head -8
for S in 0 1; do
if [ $S = 1 ]; then export KAN_NO_IM2COL=1; fi
timeout -s KILL 120 python scripts/prof_layer.py --config c5 --iters 3 > /tmp/p5.log 2>&1; tail -21 /tmp/p5.log | awk -v s=$S '{t+=$3; printf "%s ", $3} END {print " no_im2col", s, "total", t}'
done
unset KAN_NO_IM2COL
timeout -s KILL 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err; tail -3 /tmp/b.err
python -c "import json;d=json.load(open('/tmp/b.json'));print('c5', d['value'],d['ms_per_step'],d['e2e'])"
