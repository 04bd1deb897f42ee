cd $GRAFT_REPO_ROOT
for sp in 1 2; do
  echo "== split $sp"; timeout -s KILL 60 python scripts/conv_probe.py 8 8 8 8 3 1 1 bspline-lut $sp 2>&1 | grep -E "OK|MISMATCH|Error" | tail -1
  echo "== split $sp 1x1"; timeout -s KILL 60 python scripts/conv_probe.py 40 8 8 8 1 1 0 bspline-lut $sp 2>&1 | grep -E "OK|MISMATCH|Error" | tail -1
  echo "== split $sp C4"; timeout -s KILL 60 python scripts/conv_probe.py 64 32 32 64 3 1 1 bspline-lut $sp 2>&1 | grep -E "OK|MISMATCH|Error" | tail -1
done
