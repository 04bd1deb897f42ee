for o in "convw_lock=0" "convw_lock=1"; do
  echo "== c5 $o"; timeout 300 python scripts/prof_layer.py --config c5 --iters 3 --opt $o | tr '\n' ' '; echo
done
for o in "convw_lock=0" "convw_lock=1"; do
  echo "== c4 $o"; timeout 300 python scripts/prof_layer.py --config c4 --iters 20 --opt $o | tr '\n' ' '; echo
done
timeout 600 python -m pytest tests/test_gpu_conv.py -m gpu -q -x -p no:cacheprovider -k "convw" 2>&1 | tail -3
