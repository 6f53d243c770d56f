for P in 0 1; do
if [ $P = 1 ]; then export DDB_TMA_PERSISTENT=1; fi
echo "== persistent=$P"
python scripts/syrk_k.py 8192 256
python scripts/syrk_k.py 4096 256
python scripts/syrk_k.py 8192 1024
python scripts/shape_time.py 7680 256 256 fast N T
python scripts/potrf_time.py 8192 256 fast
done
