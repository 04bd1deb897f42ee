python scripts/prof_layer.py --config c5 --iters 1 --batch 2048 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:convw -s 0 -c 1 -o gpurun_out/r02_c5_l1 -f python scripts/prof_layer.py --config c5 --iters 1 --batch 2048 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
tail -3 gpurun_out/ncu_full.log
