# C1/C2: split-K and batches-in-flight choices after the epilogue changes
cd $GRAFT_REPO_ROOT
for a in ${SWEEP:-"c1 1 8"}; do
  set -- $a
  timeout -s KILL 300 python bench.py --config $1 --split-k $2 --streams $3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 split $2 streams $3', round(d['ms_per_step']*1e3,2), 'us', d['clocks']['sm_mhz'])"
done
