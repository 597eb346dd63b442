# A/B ablations of the 3xF16C pair kernel (timing only)
K=igemm_3xf16:64:2:h32,igemm_3xf16:128:2,igemm_3xf16:256:2
L=res2_3x3,res3_3x3_s2,res3_3x3,res4_3x3
echo "== base"; timeout 300 python scripts/probe_tc.py --n 256 --layers $L --kinds $K --reps 10 2>&1 | grep -v "^\s*$" | grep "ms"
for v in noconv noepi mma1; do
  echo "== $v"; CONVIO_LIB=paper_2012_15667_b200/lib/variants/$v/libconvio_b200.so timeout 300 python scripts/probe_tc.py --n 256 --layers $L --kinds $K --reps 10 2>&1 | grep "ms"
done
