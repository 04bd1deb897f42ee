set -x
KAN_EXTRA_NVFLAGS="-DKAN_TUNING" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/abl_build.log 2>&1
for r in 232 332 432 422 442; do
  echo "rings $r"; python scripts/prof_layer.py --config c5 --batch 2048 --iters 3 --opt dbg_flags=426 --opt convw_rings=$r 2>&1 | grep -E "layer (1|7|12|17):"
done
python scripts/prof_layer.py --config c5 --iters 1 > gpurun_out/plain5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/r02_launches_prof.csv python scripts/prof_layer.py --config c5 --iters 1 > /dev/null 2>&1; echo "ncu rc=$?"
