cd $GRAFT_REPO_ROOT
for c in c3bf16 c3; do
 for v in "" "KAN_FORCE_BN=128" "KAN_FORCE_BN=128 KAN_FORCE_NACC1=1" "KAN_FORCE_NACC1=1"; do env $v timeout -s KILL 300 python scripts/prof_layer.py --config $c --iters 3 2>&1 | tail -4 | head -2 | tr '\n' ' ' | sed "s/^/$c [$v]: /"; echo; done
done
