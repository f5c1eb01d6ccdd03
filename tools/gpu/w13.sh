mkdir -p gpurun_out/w13
for t in 384 192 256 512 768; do echo "== trans_min $t"; WHEELSIEVE_TRANS_MIN=$t python tools/prof_run.py c3s 3 2>&1 | tail -1; done | tee gpurun_out/w13/transmin.log
for l in 1024 1280 1536; do echo "== wc limit $l"; WHEELSIEVE_WIDE_WC_LIMIT=$l python tools/prof_run.py c3s 3 2>&1 | tail -1; done | tee gpurun_out/w13/wclimit.log
for k in 32768 49152 65536; do echo "== skip5 $k"; WHEELSIEVE_WIDE_SKIP5=$k python tools/prof_run.py c3s 3 2>&1 | tail -1; done | tee gpurun_out/w13/skip5.log
