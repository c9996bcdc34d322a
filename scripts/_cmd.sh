O=gpurun_out; mkdir -p $O
for x in "" "-DMRRR_ZG=4" "-DMRRR_FC_MINB=8" "-DMRRR_ZG=4 -DMRRR_FC_MINB=8" "-DMRRR_ZG=16"; do
MRRR_NVCC_EXTRA="$x" python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for w in C2 C5a; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 --workload $w | python scripts/bench_summary.py $w "[$x]"; done
done
