"""Ablation builds of the yzt forward kernel (diagnostics only): copy csrc/ to
a temp dir, disable one stage's work in dft_fwd_tc.cu (results become wrong,
the pipeline hand-offs stay intact), build lib/variants/libdfno_<name>.so.
Timing them (tools/ab_time.sh) shows which stage bounds the kernel.
usage: python tools/ablate_fwd.py"""
import re
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2211_12709_b200 import build as B  # noqa: E402

SRC = B.CSRC / "dft_fwd_tc.cu"

ABLATIONS = {
    # stage-T MMAs not issued (commits still signal the hand-offs)
    "noT": [(r"tc::mma_tf32_ts\(d, a \+ 32 \+ 8 \* s, bh, id, \(tb \| s\) \? 1u : 0u\);", ""),
            (r"tc::mma_tf32_ts\(d, a \+ 8 \* s, bl, id, 1u\);", ""),
            (r"tc::mma_tf32_ts\(d, a \+ 8 \* s, tc::desc\(sbt \+ \(uint32_t\)\(tb \* 4 \+ s\) \* 256, 128, L.sbo_t\), id, 1u\);", "")],
    "noZ": [(r"tc::mma_tf32_ts\(d, a \+ 8 \* s, bb, id64, \(gi.zb \| s\) \? 1u : 0u\);", ""),
            (r"tc::mma_tf32_ts\(d \+ 32, a \+ 32 \+ 8 \* s, bb, id32, 1u\);", "")],
    "noY": [(r"tc::mma_tf32\(d, ah, bh, id, \(yc \| s\) \? 1u : 0u\);", ""),
            (r"tc::mma_tf32\(d, al, bh, id, 1u\);", ""), (r"tc::mma_tf32\(d, ah, bl, id, 1u\);", "")],
    # T epilogue: no transpose / split / A_Z store (load D1, release, signal)
    "noTepi": [(r"for \(int part = 0; part < 2; \+\+part\) \{  // A_Z cols", "for (int part = 0; part < 0; ++part) {  // A_Z cols")],
    # converters: no activation math (raw copy + split)
    "noAct": [(r"return act_apply2<ACT>\(v\);", "return v;")],
}


def main():
    base = SRC.read_text()
    out = B.LIBDIR / "variants"
    out.mkdir(parents=True, exist_ok=True)
    for name, edits in ABLATIONS.items():
        txt = base
        for pat, rep in edits:
            txt, n = re.subn(pat, rep, txt)
            if n == 0:
                raise SystemExit(f"{name}: pattern not found: {pat}")
        tmp = Path(tempfile.mkdtemp())
        shutil.copytree(B.CSRC, tmp / "csrc")
        (tmp / "csrc" / "dft_fwd_tc.cu").write_text(txt)
        objs = []
        for src in sorted((tmp / "csrc").glob("*.cu")):
            obj = tmp / (src.stem + ".o")
            cmd = [B.nvcc(), *B.ARCH, *[f if not f.startswith(f"-I{B.CSRC}") else f"-I{tmp / 'csrc'}" for f in B.NVCC_FLAGS],
                   "-c", str(src), "-o", str(obj)]
            objs.append((cmd, obj))
        procs = [subprocess.Popen(c, stdout=subprocess.PIPE, stderr=subprocess.PIPE) for c, _ in objs]
        for p in procs:
            if p.wait():
                raise SystemExit(p.stderr.read().decode())
        lib = out / f"libdfno_{name}.so"
        subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(lib), *[str(o) for _, o in objs], "-lcudart"], check=True)
        shutil.rmtree(tmp)
        print(lib)


if __name__ == "__main__":
    main()
