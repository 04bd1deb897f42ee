cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
timeout -s KILL 200 python scripts/prof_layer.py --config c5 --iters 2 --nograph --batch 8192 > gpurun_out/prof/plain_c5.log 2>&1; echo PLAIN $?
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:kan_conv3 -s 3 -c 1 -o gpurun_out/prof/c5_l4 python scripts/prof_layer.py --config c5 --iters 2 --nograph --batch 8192 > gpurun_out/prof/ncu_c5.log 2>&1; echo NCU $?
