# A/B of two builds of libkan_b200.so on one box (alt/libkan_b200_old.so vs the current build)
cd $GRAFT_REPO_ROOT
L=paper_2603_17230_b200/libkan_b200.so
cp $L paper_2603_17230_b200/alt/libkan_b200_new.so
for i in $(seq ${AB_REPS:-3}); do
 for v in ${AB_VARIANTS:-new old}; do
  cp paper_2603_17230_b200/alt/libkan_b200_$v.so $L
  for c in ${AB_CONFIGS:-c2 c1}; do
   timeout -s KILL 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$c', round(d['ms_per_step']*1e3,2), 'us', d['clocks']['sm_mhz'])"
  done
 done
done
cp paper_2603_17230_b200/alt/libkan_b200_new.so $L
