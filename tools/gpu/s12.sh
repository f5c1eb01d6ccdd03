for c in c5 c4; do
  for bud in 8589934592 4294967296 2147483648 1073741824; do
    for ctas in 0 2; do echo "== $c budget=$bud ctas=$ctas"; WHEELSIEVE_BUCKET_BUDGET=$bud WHEELSIEVE_BUCKET_CTAS=$ctas python tools/prof_run.py $c 3 2>&1 | tail -1; done
  done
done
