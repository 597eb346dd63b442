P="timeout 300 python scripts/probe_tc.py --n 256 --layers res2_3x3,res3_3x3_s2,res4_3x3_s2,res5_3x3_s2 --kinds igemm_3xtf32:64:2:h32,igemm_3xtf32:128:2,igemm_3xtf32:256:2,igemm_3xtf32:128:4"
timeout 300 python scripts/probe_wtc_chunk.py --layer res3_3x3 --z 128 --nzt 4 --e 4 --sweep 32768 2>&1 | grep res3
cp paper_2012_15667_b200/lib/exp/libexp.so paper_2012_15667_b200/lib/libconvio_b200.so
echo "== no B conversion (wrong numerics, timing bound)"
$P 2>&1 | grep res
timeout 300 python scripts/probe_wtc_chunk.py --layer res4_3x3 --z 256 --nzt 2 --e 4 --sweep 32768 2>&1 | grep res4
timeout 300 python scripts/probe_wtc_chunk.py --layer res3_3x3 --z 128 --nzt 4 --e 4 --sweep 32768 2>&1 | grep res3
