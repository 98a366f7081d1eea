"""Build a variant of libballmatch_b200.so with extra nvcc -D flags (A/B experiments):
  python tools/build_variant.py NAME -DBMB_PF_MASK=3 ...  ->  build/variants/NAME.so
Load it with BMB_LIB=build/variants/NAME.so (paper_2509_01180_b200/_lib.py)."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2509_01180_b200 import build as B  # noqa: E402


VARIANT_SOURCES = ("refine.cu", "expand_factored.cu", "seed.cu")


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out_dir = ROOT / "build" / "variants"
    obj_dir = out_dir / name
    obj_dir.mkdir(parents=True, exist_ok=True)
    B.build()
    objs = []
    for src in B.sources():
        obj = B.OBJ / (src.name + ".o")
        if src.name in VARIANT_SOURCES:
            obj = obj_dir / (src.name + ".o")
            cmd = [B.NVCC, *B.ARCH, *B.CFLAGS, *defs, "-c", str(src), "-o", str(obj)]
            subprocess.run(cmd, check=True)
        objs.append(str(obj))
    lib = out_dir / f"{name}.so"
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", str(lib), *objs, *B.LIBS], check=True)
    print(lib)


if __name__ == "__main__":
    main()
