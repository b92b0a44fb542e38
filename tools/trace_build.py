"""Instrumented build for phase timelines: compiles csrc/ with -DSG_TRACE (the flash
kernels' SG_TR clock64() stamps, read back by sg_debug_trace / tools/ftrace.py) and
patches a copy of csrc/sg_gemm.cu (GEMM epilogue / MMA warps, tools/gtrace.py), linked
into paper_2104_05343_b200/libsg_trace.so (selected through SG_LIB_PATH). The product
library is untouched.

    python tools/trace_build.py
"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CSRC = ROOT / "paper_2104_05343_b200" / "csrc"
OUT = ROOT / "paper_2104_05343_b200" / os.environ.get("SG_TRACE_OUT", "libsg_trace.so")
TMP = Path("/tmp/sg_trace" + os.environ.get("SG_TRACE_OUT", ""))
NVCC = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
        "-DSG_TRACE", *os.environ.get("SG_TRACE_DEFS", "").split(),
        "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", f"-I{CSRC}"]


def patch(src: str, edits) -> str:
    for old, new in edits:
        if src.count(old) != 1:
            sys.exit(f"trace patch anchor not found exactly once: {old[:70]!r}")
        src = src.replace(old, new)
    return src


GEMM = [
    ("constexpr int kBM = 128;\nconstexpr int kBK = 64;",
     "constexpr int kBM = 128;\nconstexpr int kBK = 64;\n__device__ unsigned long long g_gtrace[4][4096];\n"
     "__device__ __forceinline__ void gtr(int which, int& i, int ev) {\n"
     "  if (i < 4096) g_gtrace[which][i++] = ((unsigned long long)ev << 56) | (clock64() & 0xffffffffffffffull);\n}"),
    ("      mbar_wait_sleep(&tfull[as], aph);", "      if (trg) gtr(0, tri, 0);\n      mbar_wait_sleep(&tfull[as], aph);\n      if (trg) gtr(0, tri, 1);"),
    ("        uint32_t r[32];\n        tmem_ld32(tacc + c * 32, r);\n        tmem_wait_ld();\n",
     "        uint32_t r[32];\n        if (trg) gtr(0, tri, 2);\n        tmem_ld32(tacc + c * 32, r);\n        tmem_wait_ld();\n"
     "        if (trg) gtr(0, tri, 3);\n"),
    ("          if (in_kind) {\n            mbar_wait(&inbar[e * 2 + si], (inph >> si) & 1);\n            inph ^= 1u << si;\n          }\n",
     "          if (trg) gtr(0, tri, 4);\n          if (in_kind) {\n            mbar_wait(&inbar[e * 2 + si], (inph >> si) & 1);\n"
     "            inph ^= 1u << si;\n          }\n          if (trg) gtr(0, tri, 5);\n"),
    ("            __syncwarp();  // every lane has consumed the staged inputs before D overwrites them",
     "            if (trg) gtr(0, tri, 6);\n            __syncwarp();  // every lane has consumed the staged inputs before D overwrites them"),
    ("    bool pref_next = false;  // the next tile's first chunk input is in flight",
     "    bool pref_next = false;  // the next tile's first chunk input is in flight\n"
     "    const bool trg = blockIdx.x == 0 && e == 0 && lane == 0;\n    int tri = 0;"),
    ('extern "C" int sg_gemm(const sg_gemm_args* a, void* stream) {',
     'extern "C" int sg_debug_gtrace(void* host) {\n'
     "  return cudaMemcpyFromSymbol(host, sg::g_gtrace, sizeof(sg::g_gtrace)) == cudaSuccess ? 0 : 1;\n}\n"
     'extern "C" int sg_gemm(const sg_gemm_args* a, void* stream) {'),
    ("        if (PAIR)\n          mbar_wait_cluster(&tempty[as], aph ^ 1);  // both CTAs' epilogues drained this buffer\n"
     "        else\n          mbar_wait(&tempty[as], aph ^ 1);",
     "        if (blockIdx.x == 0 && lane == 0) gtr(1, trm, 10);\n        if (PAIR)\n"
     "          mbar_wait_cluster(&tempty[as], aph ^ 1);  // both CTAs' epilogues drained this buffer\n"
     "        else\n          mbar_wait(&tempty[as], aph ^ 1);\n        if (blockIdx.x == 0 && lane == 0) gtr(1, trm, 11);"),
    ("      uint32_t stage = 0, phase = 0, it = 0;\n      for (int u = u0; u < ucount; u += ustep, ++it) {",
     "      uint32_t stage = 0, phase = 0, it = 0;\n      int trm = 0;\n"
     "      for (int u = u0; u < ucount; u += ustep, ++it) {"),
]


def main():
    TMP.mkdir(parents=True, exist_ok=True)
    objs = []
    for src in sorted(CSRC.glob("*.cu")):
        text = src.read_text()
        if src.name == "sg_gemm.cu":
            text = patch(text, GEMM)
        dst = TMP / src.name
        dst.write_text(text)
        obj = TMP / (src.stem + ".o")
        subprocess.run(NVCC + ["-c", str(dst), "-o", str(obj)], check=True)
        objs.append(str(obj))
    subprocess.run(NVCC[:3] + ["-shared", "-o", str(OUT), *objs, "-lcudart_static", "-ldl", "-lpthread", "-lrt"],
                   check=True)
    print(f"built {OUT}")


if __name__ == "__main__":
    main()
