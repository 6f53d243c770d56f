mkdir -p gpurun_out
python scripts/potrf_once.py 8192 256 fast > gpurun_out/s12_plain.log 2>&1; tail -1 gpurun_out/s12_plain.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s12_potrf_launches.csv python scripts/potrf_once.py 8192 256 fast > gpurun_out/s12_ncu.log 2>&1; echo "ncu rc=$?"
python scripts/launch_summary.py gpurun_out/s12_potrf_launches.csv | head -16
