"""Input grids for the model-parity golden fixture (shared by generator and test).

Shapes are the BASELINE.json layers (ResNet-50 / VGG-16 3x3, MobileNet /
SqueezeNet tuner layers) plus the reference tests' own small cases.  The
B200 machine model is ``s_sm = 228 KiB / 4 B``, ``n_p = 148 SMs x 2``,
``s = n_p * s_sm / 2``.
"""

B200_HW = {"s": 8638464, "s_sm": 58368, "n_p": 296}
SB_B200 = 29184  # per-block fast memory S_b = s_sm / 2 words


def L(out, cin, ker=(3, 3), stride=1, n=1):
    return {"out": list(out), "cin": cin, "ker": list(ker), "stride": stride, "n": n}


# (w_out, h_out, c_out), c_in, kernel, stride
LAYERS = {
    "resnet_c2": L((56, 56, 64), 64),
    "resnet_c3s2": L((28, 28, 128), 128, stride=2),
    "resnet_c3": L((28, 28, 128), 128),
    "resnet_c4": L((14, 14, 256), 256),
    "resnet_c5": L((7, 7, 512), 512),
    "vgg_1_1": L((224, 224, 64), 3),
    "vgg_2_2": L((112, 112, 128), 128),
    "vgg_4_2": L((28, 28, 512), 512),
    "vgg_5_1": L((14, 14, 512), 512),
    "alexnet_c1": L((55, 55, 96), 3, ker=(11, 11), stride=4),
    "mobilenet_pw": L((112, 112, 64), 32, ker=(1, 1)),
    "squeeze_fire2_e3": L((55, 55, 64), 16),
    "small_a": L((6, 6, 4), 2),
    "small_b": L((8, 8, 16), 32),
    "small_c": L((4, 4, 2), 8),
    "small_batch": L((4, 4, 2), 2, n=3),
}


def _bound_cases():
    out = []
    for name, lay in LAYERS.items():
        for s in (64, 1024, SB_B200, 8638464):
            out.append({**lay, "name": name, "alg": "direct", "s": s})
            if lay["ker"] == [3, 3] and lay["stride"] == 1:
                for e in (2, 4, 3):
                    out.append({**lay, "name": name, "alg": "winograd", "e": e, "r": 3, "s": s})
    return out


BOUND_CASES = _bound_cases()

T_CASES = (
    [{"alg": "direct", "R": R, "s": s} for R in ("1", "9/4", "9", "121/16")
     for s in (1, 2, 7, 33, 64, 65, 144, 300)]
    + [{"alg": "winograd", "e": e, "r": r, "s": s, "variant": v}
       for e, r in ((2, 3), (4, 3), (3, 3), (2, 2)) for s in (1, 3, 16, 40)
       for v in (False, True)]
    + [{"alg": "winograd", "e": 2, "r": 3, "s": s} for s in (65, 90)]
)

HWS = [B200_HW, {"s": 144}, {"s": 4096}, {"s": 96}, {"s": 512, "n_p": 4},
       {"s": 8, "s_sm": 64, "n_p": 16}]


def _tile_cases():
    out = []
    for name, lay in LAYERS.items():
        for hw in HWS:
            out.append({**lay, "name": name, "alg": "direct", "hw": hw})
            if lay["ker"] == [3, 3] and lay["stride"] == 1:
                for e in (2, 4):
                    out.append({**lay, "name": name, "alg": "winograd", "e": e, "r": 3, "hw": hw})
    return out


TILE_CASES = _tile_cases()


def T(x, y, z, s_b, nx=1, ny=1, nz=1, layout="CHW", e=None):
    return {"x": x, "y": y, "z": z, "s_b": s_b, "n_xt": nx, "n_yt": ny, "n_zt": nz,
            "layout": layout, "e": e}


SIM_CASES = [
    {**LAYERS["resnet_c2"], "alg": "direct", "hw": B200_HW, "tile": T(1, 8, 1, 47)},
    {**LAYERS["resnet_c2"], "alg": "direct", "hw": B200_HW, "tile": T(8, 28, 32, 16384, 2, 7, 4)},
    {**LAYERS["resnet_c2"], "alg": "direct", "hw": B200_HW, "tile": T(56, 4, 64, 16384, 7, 4, 8)},
    {**LAYERS["resnet_c2"], "alg": "direct", "hw": B200_HW, "tile": T(8, 8, 8, 100)},
    {**LAYERS["resnet_c3s2"], "alg": "direct", "hw": B200_HW, "tile": T(28, 4, 64, 16384, 7, 4, 8)},
    {**LAYERS["resnet_c5"], "alg": "direct", "hw": B200_HW, "tile": T(7, 7, 64, 16384, 1, 7, 8)},
    {**LAYERS["vgg_1_1"], "alg": "direct", "hw": B200_HW, "tile": T(32, 8, 64, 16384, 4, 8, 8)},
    {**LAYERS["alexnet_c1"], "alg": "direct", "hw": B200_HW, "tile": T(5, 5, 32, 8192)},
    {**LAYERS["small_a"], "alg": "direct", "hw": {"s": 144}, "tile": T(6, 6, 4, 244)},
    {**LAYERS["small_a"], "alg": "direct", "hw": {"s": 144}, "tile": T(5, 6, 4, 244)},
    {**LAYERS["small_batch"], "alg": "direct", "hw": {"s": 512}, "tile": T(4, 4, 2, 512)},
    {**LAYERS["resnet_c2"], "alg": "winograd", "e": 2, "r": 3, "hw": B200_HW,
     "tile": T(2, 4, 1, 114, e=2)},
    {**LAYERS["resnet_c2"], "alg": "winograd", "e": 2, "r": 3, "hw": B200_HW,
     "tile": T(8, 8, 32, 20000, 4, 4, 4, e=2)},
    {**LAYERS["resnet_c2"], "alg": "winograd", "e": 2, "r": 3, "hw": B200_HW,
     "tile": T(8, 8, 32, 20000, 4, 4, 4, e=2), "shared": True},
    {**LAYERS["resnet_c4"], "alg": "winograd", "e": 2, "r": 3, "hw": B200_HW,
     "tile": T(14, 14, 8, 16384, e=2), "shared": True},
    {**LAYERS["vgg_4_2"], "alg": "winograd", "e": 4, "r": 3, "hw": B200_HW,
     "tile": T(4, 28, 16, 29000, e=4), "shared": True},
    {**LAYERS["small_c"], "alg": "winograd", "e": 2, "r": 3, "hw": {"s": 512},
     "tile": T(4, 4, 2, 304, e=2)},
    {**LAYERS["small_c"], "alg": "winograd", "e": 2, "r": 3, "hw": {"s": 512},
     "tile": T(3, 4, 2, 304, e=2)},
]

SPACE_CASES = [
    {**LAYERS["resnet_c2"], "alg": "direct", "hw": B200_HW, "threads": False},
    {**LAYERS["resnet_c2"], "alg": "direct", "hw": B200_HW, "threads": True},
    {**LAYERS["resnet_c2"], "alg": "winograd", "e": 2, "r": 3, "hw": B200_HW, "threads": False},
    {**LAYERS["resnet_c4"], "alg": "winograd", "e": 2, "r": 3, "hw": B200_HW, "threads": True},
    {**LAYERS["vgg_4_2"], "alg": "winograd", "e": 4, "r": 3, "hw": B200_HW, "threads": False},
    {**LAYERS["resnet_c3s2"], "alg": "direct", "hw": B200_HW, "threads": False},
    {**LAYERS["mobilenet_pw"], "alg": "direct", "hw": B200_HW, "threads": False},
    {**LAYERS["squeeze_fire2_e3"], "alg": "direct", "hw": B200_HW, "threads": False},
    {**LAYERS["alexnet_c1"], "alg": "direct", "hw": B200_HW, "threads": False},
    {**LAYERS["small_b"], "alg": "direct", "hw": {"s": 4096, "s_sm": 2048}, "threads": True},
]

TUNE_CASES = [
    {**L((2, 2, 2), 2), "alg": "direct", "hw": {"s": 256, "s_sm": 128}, "budget": 12,
     "seed": 7, "n_s": 4},
    {**LAYERS["small_b"], "alg": "direct", "hw": {"s": 4096, "s_sm": 2048}, "budget": 40,
     "seed": 1, "n_s": 8},
    {**LAYERS["small_b"], "alg": "direct", "hw": {"s": 4096, "s_sm": 2048}, "budget": 40,
     "seed": 2, "n_s": 8, "patience": 2},
    {**LAYERS["resnet_c2"], "alg": "direct", "hw": B200_HW, "budget": 48, "seed": 0, "n_s": 16},
    {**LAYERS["resnet_c4"], "alg": "winograd", "e": 2, "r": 3, "hw": B200_HW, "budget": 32,
     "seed": 3, "n_s": 8},
]

ORACLE_CASES = [
    {**LAYERS["small_b"], "alg": "direct", "hw": {"s": 4096, "s_sm": 2048}, "threads": True,
     "budget": 50, "seed": 4},
    {**LAYERS["resnet_c2"], "alg": "direct", "hw": B200_HW, "threads": False,
     "budget": 64, "seed": 5},
    {**LAYERS["resnet_c4"], "alg": "winograd", "e": 2, "r": 3, "hw": B200_HW,
     "threads": False, "budget": 64, "seed": 6},
]
