set -x
KAN_EXTRA_NVFLAGS="-DKAN_TUNING" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/abl_build.log 2>&1
for f in "$@"; do
  echo "opt $f"; python scripts/prof_layer.py --config c5 --batch 2048 --iters 3 --opt $f 2>&1 | grep -v "^  " | tail -22
done
