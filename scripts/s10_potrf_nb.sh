for SP in 1 2; do echo "== DDB_SPLIT=$SP"; DDB_SPLIT=$SP timeout 300 python scripts/potrf_time.py 8192 256,384,512,768,1024 fast 2>&1 | grep -v "^$" | tail -5; done
