mkdir -p gpurun_out
python scripts/syrk_once.py 8192 > gpurun_out/s4_syrk_plain.log 2>&1; tail -1 gpurun_out/s4_syrk_plain.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4_syrk_launches.csv python scripts/syrk_once.py 8192 > gpurun_out/s4_syrk_ncu.log 2>&1; echo "ncu rc=$?"
python scripts/launch_summary.py gpurun_out/s4_syrk_launches.csv 2>&1 | head -20
