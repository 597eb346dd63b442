for v in old new old new; do
  cp paper_2012_15667_b200/lib/exp/lib$v.so paper_2012_15667_b200/lib/libconvio_b200.so
  timeout 300 python scripts/probe_tc.py --n 256 --layers res2_3x3,res4_3x3_s2 --kinds igemm_3xtf32:64:2:h32,igemm_3xtf32:256:2 2>&1 | grep res | sed "s/^/$v /"
done
cp paper_2012_15667_b200/lib/exp/libnew.so paper_2012_15667_b200/lib/libconvio_b200.so
