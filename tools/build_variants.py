"""Build A/B variants of libpetto_b200.so with different fused-kernel knobs.

    python tools/build_variants.py "W7:-DE3_W=7" "W11T:-DE3_W=11 -DE3_S=4 -DE3_TOP_SMEM=1"

Each variant goes to paper_2509_06971_b200/lib/variants/libpetto_<name>.so and its
ptxas register/spill line for k_elastic3d_fast<1> is printed.  tools/gpu_ab.sh
benches every variant on the GPU (PETTO_B200_LIB selects the library).
"""
import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_06971_b200 import build as B  # noqa: E402

OUT = os.path.join(ROOT, "paper_2509_06971_b200", "lib", "variants")


def one(spec):
    name, flags = spec.split(":", 1)
    out = os.path.join(OUT, f"libpetto_{name}.so")
    cmd = [B.nvcc()] + B.NVCC_FLAGS + flags.split() + ["-o", out, os.path.join(B.CSRC, "petto_dev.cu")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        return f"{name}: FAILED\n{r.stderr[-2000:]}"
    out = []
    for m in re.finditer(r"Compiling entry function '\S*k_elastic3d_fastILi(\d)ELb(\d)E.*?\n(?:.*?\n)*?(.*?spill.*?)\n.*?Used (\d+) registers", r.stderr):
        out.append(f"<{m.group(1)},{m.group(2)}> {m.group(4)} regs {m.group(3).strip()}")
    return f"{name}: " + ("; ".join(out) if out else "built")


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    for f in os.listdir(OUT):  # keep_* libraries (a frozen baseline) survive rebuilds
        if not f.startswith("libpetto_keep_"):
            os.remove(os.path.join(OUT, f))
    with ThreadPoolExecutor(4) as ex:
        for line in ex.map(one, sys.argv[1:]):
            print(line)
