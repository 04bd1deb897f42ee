cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
timeout -s KILL 600 python -m pytest tests -m gpu -q -x --timeout 60 --timeout-method=thread -p no:cacheprovider > /tmp/tall.log 2>&1; echo PYTEST $?; tail -1 /tmp/tall.log | cut -c1-200
# launch lists through the bench itself (graph replay), after the plain run exits 0
for cfg in c2 c4; do
  timeout -s KILL 300 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline > /tmp/plain_$cfg.json 2>/dev/null && \
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches_$cfg.csv python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "LAUNCH $cfg $?"
done
# full captures of the dominant kernels (single-GPU, one launch each)
cap() { # name config skip extra
  timeout -s KILL 200 python scripts/prof_layer.py --config $2 --iters 2 --nograph $4 > /dev/null 2>&1 && \
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:kan_gather -s $3 -c 1 -o gpurun_out/prof/$1 python scripts/prof_layer.py --config $2 --iters 2 --nograph $4 > /dev/null 2>&1; echo "CAP $1 $?"
}
cap c2_l0 c2 2 ""
cap c3_l0 c3 3 ""
cap c4_conv c4 1 ""
cap c5_l1 c5 22 "--batch 1024"
