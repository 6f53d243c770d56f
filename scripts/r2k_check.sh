set -u
mkdir -p gpurun_out
start=$(date +%s)
timeout 1200 python bench.py > gpurun_out/r2k_bench.log 2>&1; echo "bench rc=$? $(( $(date +%s) - start ))s"
tail -1 gpurun_out/r2k_bench.log | cut -c1-3000
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2k_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r2k_ref.log | cut -c1-400
