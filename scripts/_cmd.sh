O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python bench.py > $O/final_bench_C2.log 2>&1; echo "bench rc=$?"
