cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for s in 1 2 4 7; do echo "split $s"; timeout -s KILL 120 python scripts/prof_layer.py --config c2 --split $s; done
for b in 128 1024 16384; do echo "batch $b"; timeout -s KILL 120 python scripts/prof_layer.py --config c2 --batch $b --split 1; done
timeout -s KILL 120 python scripts/prof_layer.py --config c2 > gpurun_out/plain_prof.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:kan_gather -s 2 -c 1 -o gpurun_out/prof_c2_l0 python scripts/prof_layer.py --config c2 > gpurun_out/ncu_full.log 2>&1; echo NCU $?
tail -3 gpurun_out/ncu_full.log
