mkdir -p gpurun_out
python scripts/syrk_once.py 8192 > gpurun_out/s8_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"dd_tma|sym_fold" -c 2 -o gpurun_out/s8_prof_syrk python scripts/syrk_once.py 8192 > gpurun_out/s8_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/s8_ncu.log
