"""Build libdprt_cuda.so variants with extra -D flags into tools/variants/NAME.so (kernel experiments;
select one at run time with DPRT_CUDA_LIB=tools/variants/NAME.so).

    python tools/build_variant.py NAME -DDPRT_BEAM_MINBLOCKS=4 [...]
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2501_01628_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out = ROOT / "tools" / "variants" / f"{name}.so"
out.parent.mkdir(exist_ok=True)
cmd = [B.nvcc_path(), *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-ffp-contract=off",
       f"-I{B.INCLUDE}", "-Xptxas", "-v", *flags, "-o", str(out), *[str(B.CSRC / s) for s in B.SOURCES]]
p = subprocess.run(cmd, capture_output=True, text=True)
if p.returncode:
    sys.exit(p.stderr)
lines = p.stderr.splitlines()
for i, l in enumerate(lines):
    if "march_beam" in l and "Compiling" in l:
        print(name, lines[i + 1].strip(), "|", lines[i + 2].strip())
