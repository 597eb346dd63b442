# plan tables re-tuned through the package tuner (device_tuner.tune_layer) + config-5 sweeps on the tcgen05 domains
mkdir -p gpurun_out/tuned3
cp paper_2012_15667_b200/tuned/*.json gpurun_out/tuned3/
for n in 256 128 64 32; do
  f=gpurun_out/tuned3/b200_resnet50.json; [ $n != 256 ] && f=gpurun_out/tuned3/b200_resnet50_n$n.json
  timeout 900 python scripts/tune_layers.py --workload resnet50 --n $n --algs igemm_3xf16,winograd_tc_3xf16_e4 --out $f 2>&1 | grep -e "->" | tail -8
done
timeout 900 python scripts/tune_layers.py --workload vgg16 --n 32 --algs igemm_3xf16,winograd_tc_3xf16_e4 --out gpurun_out/tuned3/b200_vgg16.json 2>&1 | grep -e "->" | tail -10
timeout 900 python scripts/tuner_sweep.py --engine igemm_3xf16 --n 32 --budget 16 --out gpurun_out/r2_tuner_sweep_igemm_3xf16.json 2>&1 | tail -2
timeout 900 python scripts/tuner_sweep.py --engine igemm_3xtf32 --n 32 --budget 16 --out gpurun_out/r2_tuner_sweep_igemm_3xtf32.json 2>&1 | tail -2
