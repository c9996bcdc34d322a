# C3 / C4: segmented child-frame RQI threshold sweep (MRRR_SEGCHILDMIN), stats of hand-overs, then full-size parity
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/s27_build.log 2>&1 || { echo build failed; exit 1; }
for cfg in C4 C3; do
  for m in 8 1; do
    MRRR_SEGCHILDMIN=$m timeout 300 python bench.py --workload $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/s27_${cfg}_m$m.json 2> $O/s27_${cfg}_m$m.err
    echo "$cfg m=$m rc=$?"
    python - $O/s27_${cfg}_m$m.json <<'PY'
import json,sys
j=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
s=j['stats']
print(j['ms_per_step'], {k:s[k] for k in ('rqi_handover','ho_twist','ho_fixed','ho_rqc','zwin_reruns','uncertified','failed')}, j['phases_ms'])
PY
  done
done
MRRR_SEGCHILDMIN=1 timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -k "C3 or C4" > $O/s27_full.log 2>&1; echo "full rc=$?"; tail -3 $O/s27_full.log
