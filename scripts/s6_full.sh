O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/s6_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/s6_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x > $O/s6_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/s6_pytest.log
