mkdir -p gpurun_out
python scripts/dgemm_rate.py 8192 2>&1 | tee gpurun_out/split_dgemm.log
for v in 0 1 0 1; do echo "DDB_SPLIT=$v"; DDB_SPLIT=$v python scripts/shape_time.py 8192 8192 8192 fast; done 2>&1 | tee gpurun_out/split_time.log
for s in "4096 4096 4096" "2048 2048 65536"; do for v in 0 1; do echo "DDB_SPLIT=$v $s"; DDB_SPLIT=$v python scripts/shape_time.py $s fast; done; done 2>&1 | tee -a gpurun_out/split_time.log
DDB_SPLIT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fast or bound or split or route or golden" > gpurun_out/split_pytest.log 2>&1; tail -3 gpurun_out/split_pytest.log
