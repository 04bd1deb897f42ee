# A/B of alt/libkan_b200_old.so vs the current build: C4 bench and all C5 per-layer times
cd $GRAFT_REPO_ROOT
L=paper_2603_17230_b200/libkan_b200.so
cp $L paper_2603_17230_b200/alt/libkan_b200_new.so
for v in new old new old; do
  cp paper_2603_17230_b200/alt/libkan_b200_$v.so $L
  timeout -s KILL 300 python bench.py --config c4 --steps 2000 --warmup 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c4', round(d['ms_per_step']*1e3,2), 'us', d['clocks']['sm_mhz'])"
  timeout -s KILL 300 python scripts/prof_layer.py --config c5 --iters 2 2>&1 | grep -E "layer (1|2|3|4|8|9|13|14|18|19):" | sed 's/ us avg over 2//' | tr '\n' ' ' | sed "s/^/$v c5: /"; echo
done
cp paper_2603_17230_b200/alt/libkan_b200_new.so $L
