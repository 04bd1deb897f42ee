cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 200 python scripts/prof_layer.py --config c3 --batch 4096 --iters 2 --nograph > gpurun_out/plain_c3b.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:kan_gather -s 3 -c 1 -o gpurun_out/prof_c3_l0b python scripts/prof_layer.py --config c3 --batch 4096 --iters 2 --nograph > gpurun_out/ncu_c3b.log 2>&1; echo NCU $?
