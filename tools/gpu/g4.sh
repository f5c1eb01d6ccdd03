for c in c3 c5 c4; do bash tools/gpu/ab.sh "WHEELSIEVE_SINGLE_PRED=0" "WHEELSIEVE_SINGLE_PRED=1" $c 3; done 2>&1 | tee gpurun_out/g4_ab.log
