# usage: bash tools/gpu/ab.sh "ENV_A" "ENV_B" cfg [reps]  -- alternating runs, kernel times
A="$1"; B="$2"; CFG="$3"; REPS="${4:-3}"
for i in 1 2 3; do
  echo "== A ($A)"; env $A python tools/prof_run.py $CFG $REPS 2>&1 | tail -2
  echo "== B ($B)"; env $B python tools/prof_run.py $CFG $REPS 2>&1 | tail -2
done
