cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests -m gpu -q -x --timeout 60 --timeout-method=thread -p no:cacheprovider > /tmp/tall.log 2>&1; echo PYTEST $?; tail -1 /tmp/tall.log | cut -c1-200
for T in 0 1 2; do
echo "== TABLES $T"
for cfg in c4 c2; do KAN_TABLES=$T timeout -s KILL 60 python scripts/prof_layer.py --config $cfg --iters 5 2>&1 | tail -2 | tr '\n' ' '; echo; done
KAN_TABLES=$T timeout -s KILL 120 python scripts/prof_layer.py --config c5 --iters 3 > /tmp/p5.log 2>&1; tail -21 /tmp/p5.log | awk '{s+=$3; printf "%s ", $3} END {print " total", s}'
done
