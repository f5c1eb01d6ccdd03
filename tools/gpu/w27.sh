mkdir -p gpurun_out/w27
for pc in 32 64 96 128; do echo "== c4 FILL_PIECE=$pc"; WHEELSIEVE_FILL_PIECE=$pc python tools/prof_run.py c4 3 2>&1 | tail -1; done | tee gpurun_out/w27/piece.log
for hf in 32 64 128; do echo "== c4 HUGE_FROM=$hf"; WHEELSIEVE_HUGE_FROM=$hf python tools/prof_run.py c4 3 2>&1 | tail -1; done | tee -a gpurun_out/w27/piece.log
for b in 4294967296 17179869184; do echo "== c4 BUDGET=$b"; WHEELSIEVE_BUCKET_BUDGET=$b python tools/prof_run.py c4 3 2>&1 | tail -1; done | tee -a gpurun_out/w27/piece.log
