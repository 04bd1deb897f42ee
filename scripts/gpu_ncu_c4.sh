cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 100 python scripts/prof_layer.py --config c4 --iters 3 --nograph > gpurun_out/plain_c4.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:kan_gather -s 1 -c 1 -o gpurun_out/prof_c4r python scripts/prof_layer.py --config c4 --iters 3 --nograph > gpurun_out/ncu_c4.log 2>&1; echo NCU $?
