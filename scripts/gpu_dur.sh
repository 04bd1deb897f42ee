cd $GRAFT_REPO_ROOT
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/dur.csv python scripts/prof_layer.py --config c2 --iters 3 --nograph > /dev/null 2>&1; python scripts/ncu_durations.py /tmp/dur.csv
KAN_TIMELINE=1 timeout -s KILL 60 python scripts/timeline.py --config c2 2>&1 | grep -E "layer|per-CTA"
