O=gpurun_out
timeout 1500 python scripts/family_sweep.py > $O/r02_family_sweep.txt 2> $O/fam.err; echo "fam rc=$?"
timeout 900 python scripts/subset_sweep.py C2 C5a > $O/r02_subset_sweep.txt 2> $O/sub.err; echo "sub rc=$?"
