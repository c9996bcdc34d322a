O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python scripts/shard_time.py C5a 8 1 2>&1 | tail -1
MRRR_SEGTHREADS=0 timeout 600 python scripts/shard_time.py C5a 8 1 2>&1 | tail -1
MRRR_SEGTHREADS=262144 timeout 600 python scripts/shard_time.py C5a 8 1 2>&1 | tail -1
timeout 600 python scripts/shard_time.py C5a 4 1 2>&1 | tail -1
timeout 600 python scripts/shard_time.py C5a 2 1 2>&1 | tail -1
for w in C2 C5a C5b; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 --workload $w | python scripts/bench_summary.py $w; done
