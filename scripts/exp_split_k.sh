for sp in 1 2; do
export DDB_SPLIT=$sp
echo "== DDB_SPLIT=$sp"
python scripts/syrk_k.py 8192 256
python scripts/syrk_k.py 4096 256
python scripts/syrk_k.py 8192 512
python scripts/shape_time.py 7680 256 256 fast N T
python scripts/shape_time.py 2048 256 256 fast N T
python scripts/potrf_time.py 8192 256,512 fast
done
