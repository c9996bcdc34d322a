O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
bash scripts/final_bench.sh
bash scripts/final_profiles.sh
python scripts/launch_summary.py $O/launches_C2_final.csv 2>/dev/null | head -16
