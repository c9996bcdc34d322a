# deferred two-lane tails on a side stream: parity (cluster cases, full-size C3/C4, families), then C4/C3 timings
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/s29_build.log 2>&1 || { echo build failed; tail $O/s29_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_families.py tests/test_gpu_support.py -x -q -p no:cacheprovider > $O/s29_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/s29_tests.log
for cfg in C4 C3; do
  for m in 1 0; do
    MRRR_DEFER_TAIL=$m timeout 300 python bench.py --workload $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/s29_${cfg}_d$m.json 2> $O/s29_${cfg}_d$m.err
    echo "$cfg defer=$m rc=$?"
    python - $O/s29_${cfg}_d$m.json <<'PY'
import json,sys
j=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(j['ms_per_step'], j['phases_ms']['clusters'], j['stats']['rqi_iters'], j['gpu_launches'])
PY
  done
done
