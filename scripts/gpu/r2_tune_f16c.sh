# re-tune the plan tables with the 3xF16 implicit GEMM as a candidate; results in gpurun_out/tuned
mkdir -p gpurun_out/tuned
cp paper_2012_15667_b200/tuned/*.json gpurun_out/tuned/
for n in 256 128 64 32; do
  f=gpurun_out/tuned/b200_resnet50.json; [ $n != 256 ] && f=gpurun_out/tuned/b200_resnet50_n$n.json
  timeout 900 python scripts/tune_layers.py --workload resnet50 --n $n --algs igemm_3xf16 --out $f 2>&1 | grep -E "^\S|->" | tail -20
done
timeout 900 python scripts/tune_layers.py --workload vgg16 --n 32 --algs igemm_3xf16 --out gpurun_out/tuned/b200_vgg16.json 2>&1 | grep -e "->" | tail -20
