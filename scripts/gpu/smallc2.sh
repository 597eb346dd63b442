timeout 600 python -m pytest tests/test_conv_gpu.py -q -x -k "small_c or direct" 2>&1 | grep -E "^E  |FAILED|Error" | head -8
cat > /tmp/sc.py <<'PY'
import torch, sys
sys.path.insert(0, '.')
from paper_2012_15667_b200 import conv as C, TileConfig
x = C.to_layout(torch.rand(32, 3, 224, 224, device="cuda"), "HWC")
w = torch.rand(64, 3, 3, 3, device="cuda")
wp = C.pack_filter_direct(w)
t = TileConfig(16, 16, 32, 32768, 1, 1, 1, layout="HWC")
for _ in range(3):
    C.conv_direct(x, w, padding=1, tile=t, w_packed=wp)
torch.cuda.synchronize()
PY
timeout 300 ncu --set full --import-source on --clock-control none -k regex:smallc -c 1 -o gpurun_out/ncu_smallc -f python /tmp/sc.py > /dev/null 2>&1
ls gpurun_out/ncu_smallc*
