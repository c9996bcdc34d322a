#!/bin/bash
# One GPU session: parity tests, smoke, bench, ncu launch list + full capture of the top kernels.
# usage: bash scripts/gpu_round.sh [tag] [workload]
TAG=${1:-r01}
WL=${2:-C2}
O=gpurun_out
mkdir -p $O
nvidia-smi > $O/nvidia_smi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -20 $O/build_$TAG.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke_$TAG.log
timeout 900 python bench.py --workload $WL > $O/bench_${WL}_$TAG.log 2>&1; echo "bench rc=$?"; tail -c 3000 $O/bench_${WL}_$TAG.log
timeout 300 python scripts/profile_solve.py $WL 2 > $O/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_${WL}_$TAG.csv \
    python scripts/profile_solve.py $WL 2 > $O/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_rqi2|k_negcount|k_zwrite_chunk" -s 0 -c 4 \
    -o $O/prof_${WL}_$TAG python scripts/profile_solve.py $WL 1 > $O/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
