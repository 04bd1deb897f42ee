cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pp
for c in c2 c1; do
 for m in none 0; do
  if [ $m = none ]; then unset KAN_LEVEL_PREPASS_MIN; else export KAN_LEVEL_PREPASS_MIN=$m; fi
  timeout -s KILL 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/pp/${c}_$m.json 2>gpurun_out/pp/${c}_$m.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/pp/${c}_$m.json').read().strip().splitlines()[-1]); print('$c', '$m', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
 done
done
unset KAN_LEVEL_PREPASS_MIN
