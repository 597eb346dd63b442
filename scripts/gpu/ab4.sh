for v in head exp head exp; do
  cp paper_2012_15667_b200/lib/exp/lib$v.so paper_2012_15667_b200/lib/libconvio_b200.so
  timeout 300 python scripts/probe_tc.py --n 256 --layers res4_3x3,res4_3x3_s2,res5_3x3_s2 --kinds igemm_3xtf32:256:2 2>&1 | grep res | sed "s/^/$v /"
  timeout 300 python scripts/probe_wtc_chunk.py --layer res4_3x3 --z 256 --nzt 2 --e 4 --sweep 32768 2>&1 | grep res4 | sed "s/^/$v /"
  timeout 300 python scripts/probe_wtc_chunk.py --layer res5_3x3 --z 256 --nzt 2 --e 4 --sweep 32768 2>&1 | grep res5 | sed "s/^/$v /"
done
cp paper_2012_15667_b200/lib/exp/libhead.so paper_2012_15667_b200/lib/libconvio_b200.so
