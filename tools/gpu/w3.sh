mkdir -p gpurun_out/w3
cd tests/cpp
for w in 3 0 3 0; do
  echo "== WIDE=$w"
  WHEELSIEVE_WIDE=$w ./_ref/cli_gpu 2>&1 | grep -v "^\[PASS\]" | tail -15
done
cd ../..
for w in 3 0; do
echo "== direct WIDE=$w"
WHEELSIEVE_WIDE=$w timeout --preserve-status -s INT 1 paper_2310_17746_b200/wheelsieve sieve --limit unbounded --count-only --segment 600000; echo "rc=$?"
done
