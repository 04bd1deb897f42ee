for s in 1 2 4 8; do echo "=== c2 split $s"; python scripts/timeline.py --config c2 --split $s 2>&1 | tail -24; done
echo "=== c1 split 0"; python scripts/timeline.py --config c1 --split 0 2>&1 | tail -24
for s in 1 4; do echo "== prof c2 split $s"; python scripts/prof_layer.py --config c2 --split $s --iters 20; done
