# A/B: the previous library vs the deferred-tail library on the schedule-parity tests (same box)
O=gpurun_out
P=paper_1401_4950_b200
for v in old new; do
  cp $P/libmrrr_$v.so $P/libmrrr.so
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > $O/s32_$v.log 2>&1
  echo "$v rc=$? $(tail -1 $O/s32_$v.log)"
done
cp $P/libmrrr_new.so $P/libmrrr.so
MRRR_DEFER_TAIL=0 CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > $O/s32_blk.log 2>&1
echo "blocking rc=$?"; grep -m3 "MrrrError:" $O/s32_blk.log
