python scripts/syrk_k.py 8192 256
python scripts/syrk_k.py 4096 256
python scripts/syrk_k.py 8192 64
python scripts/syrk_k.py 8192 1024
python scripts/shape_time.py 7680 256 256 fast N T
python scripts/shape_time.py 2048 256 256 fast N T
python scripts/shape_time.py 2048 192 64 fast N N
python scripts/shape_time.py 8192 8192 8192 fast
python scripts/shape_time.py 4096 4096 4096 fast
python scripts/potrf_time.py 8192 256,512 fast
python scripts/getrf_time.py 8192 fast
