timeout 600 python scripts/f16_check.py 2>&1 | tail -20
