for c in c4 c5 c4e; do bash tools/gpu/ab.sh "WHEELSIEVE_SKIP5=0" "WHEELSIEVE_SKIP5=16384" $c 3; done 2>&1 | grep "==\|rep 2"
for c in c3s c2 c1; do echo "== $c"; python tools/prof_run.py $c 3 | tail -1; done
