# ablations of the C5 layers under a -DKAN_TUNING build (args: dbg flag values)
set -x
KAN_EXTRA_NVFLAGS="-DKAN_TUNING" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/abl_build.log 2>&1
for f in 0 "$@"; do
  echo "flags $f"; python scripts/prof_layer.py --config c5 --batch 2048 --iters 3 --opt dbg_flags=$f 2>&1 | sed -n '2,5p;8,11p'
done
