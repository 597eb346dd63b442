for v in 1 3; do
  cp paper_2012_15667_b200/lib/exp/lib$v.so paper_2012_15667_b200/lib/libconvio_b200.so
  timeout 600 python scripts/f16_check.py 2>&1 | grep -E " ms" | sed "s/^/v$v /"
done
cp paper_2012_15667_b200/lib/exp/lib1.so paper_2012_15667_b200/lib/libconvio_b200.so
