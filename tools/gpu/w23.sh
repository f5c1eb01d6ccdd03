mkdir -p gpurun_out/w23
python tools/prof_run.py c4 2 > gpurun_out/w23/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/w23/launches_c4.csv python tools/prof_run.py c4 2 > gpurun_out/w23/ncu.log 2>&1
python tools/summarize_ncu.py launches gpurun_out/w23/launches_c4.csv
python tools/prof_run.py c5 2 > gpurun_out/w23/plain5.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/w23/launches_c5.csv python tools/prof_run.py c5 2 > gpurun_out/w23/ncu5.log 2>&1
python tools/summarize_ncu.py launches gpurun_out/w23/launches_c5.csv
