# ablations of the C5 layers under a -DKAN_TUNING build (args: engine options, one run each)
set -x
KAN_EXTRA_NVFLAGS="-DKAN_TUNING" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/abl_build.log 2>&1
for f in "dbg_flags=0" "$@"; do
  echo "opt $f"; python scripts/prof_layer.py --config c5 --batch 2048 --iters 3 --opt $f 2>&1 | sed -n '2,5p;8,10p;13,15p;18,20p'
done
