O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/s30_build.log 2>&1 || exit 1
for yw in 8 128; do for dt in 1 0; do
  echo "== SEGYW=$yw DEFER=$dt"; MRRR_SEGYW=$yw MRRR_DEFER_TAIL=$dt timeout 120 python scripts/s30_dbg.py 2>&1 | tail -4
done; done
echo "== sanitizer"
MRRR_SEGYW=8 timeout 600 compute-sanitizer --print-limit 5 python scripts/s30_dbg.py > $O/s30_san.log 2>&1; echo rc=$?
grep -m 20 -E "Invalid|at 0x|by thread|Address|FAIL|ok" $O/s30_san.log
