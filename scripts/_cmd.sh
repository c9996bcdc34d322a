O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 300 python scripts/profile_solve.py C3 1 > $O/plain_C3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3.csv python scripts/profile_solve.py C3 1 > /dev/null 2>&1; python scripts/launch_summary.py $O/launches_C3.csv 2>/dev/null | head -20
