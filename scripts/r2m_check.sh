set -u
mkdir -p gpurun_out
df -h /dev/shm | tail -1
timeout 900 python bench.py --force-dist --steps 3 --warmup 3 > gpurun_out/r2m_dist.log 2>&1; echo "dist rc=$?"; tail -1 gpurun_out/r2m_dist.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps(d.get('e2e')), json.dumps(d.get('config5')))"
