./scripts/dev/umma_shift_selftest 2>&1 | grep "rate"
