"""Build an A/B experiment variant of libdfno.so with extra nvcc flags into
paper_2211_12709_b200/lib/variants/libdfno_<name>.so (the product always
loads lib/libdfno.so; tools/ab_time.sh swaps a variant in for timing only).
Usage: python tools/build_variant.py <name> -DFOO=1 ..."""
import concurrent.futures as cf
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2211_12709_b200 import build as B  # noqa: E402


def main(name, flags):
    out = B.LIBDIR / "variants"
    objdir = out / f"obj_{name}"
    objdir.mkdir(parents=True, exist_ok=True)

    def comp(src):
        obj = objdir / (src.stem + ".o")
        cmd = [B.nvcc(), *B.ARCH, *B.NVCC_FLAGS, *flags, "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise SystemExit(r.stderr)
        return obj

    srcs = B._sources()
    with cf.ThreadPoolExecutor(max_workers=8) as ex:
        objs = list(ex.map(comp, srcs))
    lib = out / f"libdfno_{name}.so"
    subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcudart"], check=True)
    print(lib)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
