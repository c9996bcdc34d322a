# re-entry check after the container was re-created: rebuild, smoke, default bench (both arms), full GPU suite
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/s35_build.log 2>&1 || exit 1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/s35_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > $O/r02f_bench_C2.json 2> $O/s35_bench.err; echo "bench rc=$?"
python bench.py --impl reference > $O/r02f_reference_C2.json 2> $O/s35_ref.err; echo "ref rc=$?"
python -m pytest tests -m gpu -x -q > $O/r02f_gpu_tests.log 2>&1; echo "gpu tests rc=$?"
tail -3 $O/r02f_gpu_tests.log
cat $O/r02f_bench_C2.json
