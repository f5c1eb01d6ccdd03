for c in c5 c4; do bash tools/gpu/ab.sh "WHEELSIEVE_FILL_UNROLL=0" "WHEELSIEVE_FILL_UNROLL=1" $c 3; done 2>&1 | grep "==\|rep 2"
