K=igemm_3xf16:64:2:h32,igemm_3xf16:128:2,igemm_3xf16:256:2,igemm_3xf16:128:2:h16
L=res2_3x3,res3_3x3_s2,res3_3x3,res4_3x3
for st in 2 3 4 6; do echo "== stages<=$st"; CONVIO_DEV_MAX_STAGES=$st timeout 300 python scripts/probe_tc.py --n 256 --layers $L --kinds $K --reps 10 2>&1 | grep " ms"; done
echo "== tmaonly"; CONVIO_LIB=paper_2012_15667_b200/lib/variants/tmaonly/libconvio_b200.so timeout 300 python scripts/probe_tc.py --n 256 --layers $L --kinds $K --reps 10 2>&1 | grep " ms"
