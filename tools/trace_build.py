"""Instrumented build for phase timelines: patches copies of csrc/sg_attn.cu (flash
backward) and csrc/sg_gemm.cu (GEMM epilogue / MMA warps) with clock64() stamps and
links paper_2104_05343_b200/libsg_trace.so (read by tools/ftrace.py, tools/gtrace.py
through SG_LIB_PATH). The product library is untouched.

    python tools/trace_build.py
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CSRC = ROOT / "paper_2104_05343_b200" / "csrc"
OUT = ROOT / "paper_2104_05343_b200" / "libsg_trace.so"
TMP = Path("/tmp/sg_trace")
NVCC = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
        "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", f"-I{CSRC}"]


def patch(src: str, edits) -> str:
    for old, new in edits:
        if src.count(old) != 1:
            sys.exit(f"trace patch anchor not found exactly once: {old[:70]!r}")
        src = src.replace(old, new)
    return src


ATTN = [
    ("constexpr uint32_t kT64 = 128 * 64 * 2;  // one 128 x 64 bf16 tile (16 KB)",
     "constexpr uint32_t kT64 = 128 * 64 * 2;  // one 128 x 64 bf16 tile (16 KB)\n"
     "__device__ unsigned long long g_ftrace[2][8192];\n"
     "__device__ __forceinline__ void ftr(int which, int& i, int ev) {\n"
     "  if (i < 8192) g_ftrace[which][i++] = ((unsigned long long)ev << 56) | (clock64() & 0xffffffffffffffull);\n}"),
    ('extern "C" int sg_flash_attn_bwd(',
     'extern "C" int sg_debug_ftrace(void* host) {\n'
     "  return cudaMemcpyFromSymbol(host, sg::g_ftrace, sizeof(sg::g_ftrace)) == cudaSuccess ? 0 : 1;\n}\n"
     'extern "C" int sg_flash_attn_bwd('),
    ("      if (total > 0) issue_sdp(0);\n      for (int G = 0; G < total; ++G) {\n"
     "        const int slot = G & 1, it = G / nqb, i = G % nqb;\n",
     "      const bool trm = blockIdx.x == 0;\n      int tri = 0;\n"
     "      if (total > 0) issue_sdp(0);\n      for (int G = 0; G < total; ++G) {\n"
     "        const int slot = G & 1, it = G / nqb, i = G % nqb;\n        if (trm) ftr(1, tri, 20);\n"),
    ("        if (G + 1 < total) issue_sdp(G + 1);\n",
     "        if (trm) ftr(1, tri, 21);\n        if (G + 1 < total) issue_sdp(G + 1);\n        if (trm) ftr(1, tri, 22);\n"),
    ("        mbar_wait(ds_full, G & 1);  // P_G, dS_G in smem\n        tc_fence_after();\n",
     "        mbar_wait(ds_full, G & 1);  // P_G, dS_G in smem\n        tc_fence_after();\n        if (trm) ftr(1, tri, 23);\n"),
    ("        umma_commit(&qd_empty[slot]);\n        if (G >= 2)",
     "        umma_commit(&qd_empty[slot]);\n        if (trm) ftr(1, tri, 24);\n        if (G >= 2)"),
    ("    int kb = 0, h = 0, b = 0;\n    if (my_items > 0) item(0, kb, h, b);\n    for (int G = 0; G < total; ++G) {\n",
     "    int kb = 0, h = 0, b = 0;\n    if (my_items > 0) item(0, kb, h, b);\n"
     "    const bool trs = blockIdx.x == 0 && e == 0 && lane == 0;\n"
     "    int tri = 0;\n    for (int G = 0; G < total; ++G) {\n      if (trs) ftr(0, tri, 0);\n"),
    ("      mbar_wait(s_full, G & 1);\n      tc_fence_after();\n",
     "      mbar_wait(s_full, G & 1);\n      tc_fence_after();\n      if (trs) ftr(0, tri, 1);\n"),
    ("      // the previous block's dV / dK / dQ products have finished reading P / dS\n",
     "      if (trs) ftr(0, tri, 4);\n      // the previous block's dV / dK / dQ products have finished reading P / dS\n"),
    ("      if (lane == 0) mbar_arrive(ds_full);\n      if (i == nqb - 1) {",
     "      if (lane == 0) mbar_arrive(ds_full);\n      if (trs) ftr(0, tri, 6);\n      if (i == nqb - 1) {"),
]

GEMM = [
    ("constexpr int kBM = 128;\nconstexpr int kBK = 64;",
     "constexpr int kBM = 128;\nconstexpr int kBK = 64;\n__device__ unsigned long long g_gtrace[4][4096];\n"
     "__device__ __forceinline__ void gtr(int which, int& i, int ev) {\n"
     "  if (i < 4096) g_gtrace[which][i++] = ((unsigned long long)ev << 56) | (clock64() & 0xffffffffffffffull);\n}"),
    ("      mbar_wait(&tfull[as], aph);", "      if (trg) gtr(0, tri, 0);\n      mbar_wait(&tfull[as], aph);\n      if (trg) gtr(0, tri, 1);"),
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
     "        if (blockIdx.x == 0) gtr(1, trm, 10);\n        if (PAIR)\n"
     "          mbar_wait_cluster(&tempty[as], aph ^ 1);  // both CTAs' epilogues drained this buffer\n"
     "        else\n          mbar_wait(&tempty[as], aph ^ 1);\n        if (blockIdx.x == 0) gtr(1, trm, 11);"),
    ("      uint32_t stage = 0, phase = 0, it = 0;\n      for (int t = unit0; t < p.num_tiles; t += nunits, ++it) {",
     "      uint32_t stage = 0, phase = 0, it = 0;\n      int trm = 0;\n"
     "      for (int t = unit0; t < p.num_tiles; t += nunits, ++it) {"),
]


def main():
    TMP.mkdir(parents=True, exist_ok=True)
    objs = []
    for src in sorted(CSRC.glob("*.cu")):
        text = src.read_text()
        if src.name == "sg_attn.cu":
            text = patch(text, ATTN)
        elif src.name == "sg_gemm.cu":
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
