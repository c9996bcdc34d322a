O=gpurun_out
python scripts/timeline.py C1 > $O/s13_timeline_C1.txt 2>&1; echo "timeline rc=$?"; head -24 $O/s13_timeline_C1.txt
python scripts/sweep_env.py C1 5 ""
python scripts/sweep_env.py C2 5 ""
