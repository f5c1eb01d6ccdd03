mkdir -p gpurun_out/w20
bash tools/gpu/ab.sh "WHEELSIEVE_SINGLE_PRED=0" "WHEELSIEVE_SINGLE_PRED=1" c3s 3 2>&1 | grep -v "rep 0\|rep 1" | head -8 | tee gpurun_out/w20/ab_pred.log
