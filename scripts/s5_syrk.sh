mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "syrk or Syrk or split or potrf" > gpurun_out/s5_pytest.log 2>&1; echo "pytest: $(tail -1 gpurun_out/s5_pytest.log)"
python scripts/syrk_once.py 8192 2>&1 | tail -1
python scripts/syrk_once.py 4096 2>&1 | tail -1
python scripts/potrf_time.py 8192 256 fast 2>&1 | tail -2
