"""Generate the explicit instantiations of the direct-conv kernel template.

The register micro-tile (TX, TY, TZ) and the kernel edge / stride must be
compile-time for the inner loop to live in registers, so the legal device
projection of a TileConfig is "its micro-tile x/n_xt, y/n_yt, z/n_zt is in
this table".  Instances are spread over several translation units so nvcc
can build them in parallel.

    python gen_instances.py OUTDIR
"""

import os
import sys

# (kernel edge, stride) -> (TX set, TY set, TZ set, max accumulators)
FAMILIES = {
    (3, 1): ((1, 2, 4, 7, 8), (1, 2, 4), (1, 2, 4, 8, 16), 128),
    (3, 2): ((1, 2, 4, 7), (1, 2), (2, 4, 8, 16), 64),
    (1, 1): ((1, 2, 4, 7, 8), (1, 2), (4, 8, 16), 128),
    (1, 2): ((1, 2, 4, 7), (1, 2), (4, 8, 16), 64),
}
N_UNITS = 8


def instances():
    out = []
    for (ks, st), (txs, tys, tzs, cap) in FAMILIES.items():
        for tx in txs:
            for ty in tys:
                for tz in tzs:
                    if tx * ty * tz <= cap:
                        out.append((ks, st, tx, ty, tz))
    return out


def main(outdir):
    os.makedirs(outdir, exist_ok=True)
    inst = instances()
    units = [inst[i::N_UNITS] for i in range(N_UNITS)]
    for u, items in enumerate(units):
        lines = ['#include "../direct_fp32.cuh"', "namespace convio {",
                 "struct DirectEntry { int ks, st, tx, ty, tz; DirectKernelFn fn; };",
                 f"extern const DirectEntry g_direct_entries_{u}[] = {{"]
        for ks, st, tx, ty, tz in items:
            lines.append(f"    {{{ks}, {st}, {tx}, {ty}, {tz}, "
                         f"&direct_conv_f32_kernel<{ks}, {st}, {tx}, {ty}, {tz}>}},")
        lines.append("    {0, 0, 0, 0, 0, nullptr}};")
        lines.append("}  // namespace convio")
        path = os.path.join(outdir, f"direct_inst_{u}.cu")
        text = "\n".join(lines) + "\n"
        if not os.path.exists(path) or open(path).read() != text:
            with open(path, "w") as fh:
                fh.write(text)
    reg = ['#include "../direct_fp32.cuh"', "namespace convio {",
           "struct DirectEntry { int ks, st, tx, ty, tz; DirectKernelFn fn; };"]
    for u in range(N_UNITS):
        reg.append(f"extern const DirectEntry g_direct_entries_{u}[];")
    reg.append("static const DirectEntry *const kUnits[] = {"
               + ", ".join(f"g_direct_entries_{u}" for u in range(N_UNITS)) + "};")
    reg.append("""DirectKernelFn find_direct_kernel(int ks, int st, int tx, int ty, int tz) {
    for (const DirectEntry *unit : kUnits)
        for (const DirectEntry *e = unit; e->fn != nullptr; ++e)
            if (e->ks == ks && e->st == st && e->tx == tx && e->ty == ty && e->tz == tz)
                return e->fn;
    return nullptr;
}""")
    reg.append(f"int direct_instance_count() {{ return {len(inst)}; }}")
    reg.append("}  // namespace convio")
    path = os.path.join(outdir, "direct_registry.cu")
    text = "\n".join(reg) + "\n"
    if not os.path.exists(path) or open(path).read() != text:
        with open(path, "w") as fh:
            fh.write(text)
    print(f"{len(inst)} direct instances in {N_UNITS} units -> {outdir}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "gen"))
