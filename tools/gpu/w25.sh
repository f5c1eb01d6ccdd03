mkdir -p gpurun_out/w25
for l in 1024 1152 1280 1408 1536; do echo "== wc limit $l"; WHEELSIEVE_WIDE_WC_LIMIT=$l python tools/prof_run.py c3s 3 2>&1 | tail -1; done | tee gpurun_out/w25/wclimit.log
for l in 1024 1280; do echo "== c4 wc limit $l"; WHEELSIEVE_WIDE_WC_LIMIT=$l python tools/prof_run.py c4 3 2>&1 | tail -1; done | tee -a gpurun_out/w25/wclimit.log
