"""Build a compile-time variant of the GPU library for A/B timing runs:
    python tools/build_variant.py NAME -DMACRO=VALUE ...
writes build/variants/NAME.so (cse.cu recompiled with the macros, the other
objects reused); select it with SPG_LIB=build/variants/NAME.so."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2005_10680_b200 import build as b  # noqa: E402

name, macros = sys.argv[1], sys.argv[2:]
b.build_gpu()
out_dir = ROOT / "build" / "variants"
out_dir.mkdir(parents=True, exist_ok=True)
obj = out_dir / f"cse_{name}.o"
subprocess.run([b.NVCC] + b.NVCC_FLAGS + macros + ["-c", str(b.CSRC / "cse.cu"), "-o", str(obj)],
               check=True)
objs = [obj if o.stem == "cse" else o for o in (b.OBJ / (Path(s).stem + ".o") for s in b.CU_SOURCES)]
subprocess.run([b.NVCC] + b.ARCH + ["-shared", "-o", str(out_dir / f"{name}.so")] + [str(o) for o in objs],
               check=True)
print(out_dir / f"{name}.so")
