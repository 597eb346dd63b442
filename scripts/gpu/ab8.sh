for v in 3 4; do
  cp paper_2012_15667_b200/lib/exp/lib$v.so paper_2012_15667_b200/lib/libconvio_b200.so
  timeout 600 python scripts/f16_check.py 2>&1 | grep -E "3xf16 .* ms" | sed "s/^/v$v /"
done
