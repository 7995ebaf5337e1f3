"""Build an A/B variant of the library: one csrc file recompiled with extra -D flags, linked with
the other current objects, written to tools/bin/<name>.so (load it with ITTS_LIB=...).

    python tools/build_variant.py NAME FILE.cu -DFOO=1 [-DBAR=2 ...]
"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2211_13939_b200 import _build  # noqa: E402

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
_build.build()
out_dir = Path(__file__).resolve().parent / "bin"
out_dir.mkdir(exist_ok=True)
obj = out_dir / f"{name}_{Path(src).stem}.o"
subprocess.run([_build.nvcc(), *_build.ARCH, *_build.BASE_FLAGS, *defs, "-c", str(_build.CSRC / src), "-o", str(obj)],
               check=True)
objs = [obj if o.stem == Path(src).stem else o for o in sorted(_build.BUILD.glob("*.o"))]
subprocess.run([_build.nvcc(), *_build.ARCH, "-shared", "-cudart", "static", "-o", str(out_dir / f"{name}.so"),
                *map(str, objs), "-lcuda"], check=True)
print(out_dir / f"{name}.so")
