"""Build a compile-time variant of the GPU library for A/B timing runs:
    python tools/build_variant.py NAME [-DMACRO=VALUE ...] [--src a.cu,b.cu]
writes build/variants/NAME.so (the given sources -- default cse.cu --
recompiled with the macros, the other objects reused); select it with
SPG_LIB=build/variants/NAME.so."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2005_10680_b200 import build as b  # noqa: E402

name, rest = sys.argv[1], sys.argv[2:]
srcs = ["cse.cu"]
macros = []
for a in rest:
    if a.startswith("--src="):
        srcs = a.split("=", 1)[1].split(",")
    else:
        macros.append(a)
b.build_gpu()
out_dir = ROOT / "build" / "variants"
out_dir.mkdir(parents=True, exist_ok=True)
objs = []
for src in b.CU_SOURCES:
    stem = Path(src).stem
    if src in srcs:
        obj = out_dir / f"{stem}_{name}.o"
        subprocess.run([b.NVCC] + b.NVCC_FLAGS + macros + ["-c", str(b.CSRC / src), "-o", str(obj)],
                       check=True)
        objs.append(obj)
    else:
        objs.append(b.OBJ / f"{stem}.o")
subprocess.run([b.NVCC] + b.ARCH + ["-shared", "-o", str(out_dir / f"{name}.so")] + [str(o) for o in objs],
               check=True)
print(out_dir / f"{name}.so")
