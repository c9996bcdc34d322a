for v in "" "-DMRRR_XG_PF=4 -DMRRR_XG_MINB=8" "-DMRRR_XG_PF=8 -DMRRR_XG_MINB=8" "-DMRRR_XG_PF=4 -DMRRR_XG_MINB=6" "-DMRRR_XG_PF=16 -DMRRR_XG_MINB=4"; do
  MRRR_NVCC_EXTRA="$v" python -c "from paper_1401_4950_b200 import _build; _build.build(force=True)" > /dev/null 2>&1 || echo "build failed $v"
  echo "== $v"
  python scripts/sweep_env.py C3 2 ""
  python scripts/sweep_env.py C4 2 ""
done
