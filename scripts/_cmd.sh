O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for v in 0 131072; do
MRRR_RQITHREADS=$v timeout 300 python scripts/shard_time.py C2 8 3 2>&1 | tail -1 | sed "s/^/RQITHREADS=$v /"
MRRR_RQITHREADS=$v timeout 300 python scripts/shard_time.py C2 2 3 2>&1 | tail -1 | sed "s/^/RQITHREADS=$v /"
MRRR_RQITHREADS=$v timeout 600 python scripts/shard_time.py C5a 8 1 2>&1 | tail -1 | sed "s/^/RQITHREADS=$v /"
done
for st in 262144 524288; do MRRR_SEGTHREADS=$st timeout 600 python scripts/shard_time.py C5a 8 1 2>&1 | tail -1 | sed "s/^/SEGTHREADS=$st /"; done
timeout 300 python scripts/shard_time.py C5a 8 1 2>&1 | head -3
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
