python scripts/timeline.py C2 2>&1 | grep -v Warn | head -30
