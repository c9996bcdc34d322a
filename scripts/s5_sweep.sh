for c in C2 C4 C5b C3; do python scripts/sweep_env.py $c 3 "MRRR_FUSEM=16" "MRRR_FUSEM=3" "MRRR_FUSEM=2" "MRRR_FUSEM=1"; done
