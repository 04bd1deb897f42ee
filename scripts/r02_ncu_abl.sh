set -x
KAN_EXTRA_NVFLAGS="-DKAN_TUNING" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/abl_build.log 2>&1
python scripts/prof_layer.py --config c5 --batch 2048 --iters 1 --opt dbg_flags=426 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:convw -s 0 -c 1 -o gpurun_out/prof_skel python scripts/prof_layer.py --config c5 --batch 2048 --iters 1 --opt dbg_flags=426 > gpurun_out/ncu_skel.log 2>&1; echo "ncu rc=$?"
