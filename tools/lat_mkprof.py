"""Copy csrc to tools/variants/src_prof with clock64 phase counters in k_lattice_idx
(then: bash tools/build_variant.sh prof tools/variants/src_prof; CTW_B200_LIB=tools/variants/lib_prof.so
python tools/lat_prof_phases.py)."""
import shutil
from pathlib import Path
R = Path(__file__).resolve().parents[1]
d = R / "tools/variants/src_prof"
shutil.rmtree(d, ignore_errors=True)
shutil.copytree(R / "paper_2311_04996_b200/csrc", d)
p = d / "ctw_lattice.cu"
S = p.read_text()
i0 = S.index("// ------------------------------------------------------------ indexed kernel")
i1 = S.index("}  // namespace\n\nextern \"C\" int ctw_launch_lattice")
s = S[i0:i1]
def rep(a, b):
    global s
    assert s.count(a) == 1, a[:70]
    s = s.replace(a, b)
rep("__global__ void __launch_bounds__(LAT_IBS, LAT_IMINB) k_lattice_idx(LatArgs a) {",
    "}  // namespace\n__device__ unsigned long long g_latprof[8];\nnamespace {\n"
    "__global__ void __launch_bounds__(LAT_IBS, LAT_IMINB) k_lattice_idx(LatArgs a) {\n"
    "  long long tA = 0, tB = 0, tC = 0, tD = 0, tE = 0, tq;")
rep("    if (sm.f < 0) break;  // the layer index lives in shared memory (no register across the layer)",
    "    if (sm.f < 0) break;\n    tq = clock64();")
rep("    // ---- destination map: nodes of layer f that can lie on a kept path",
    "    tA += clock64() - tq; tq = clock64();\n    // ---- destination map: nodes of layer f that can lie on a kept path")
rep("    __syncthreads();\n    if (sm.nmap > LAT_MAP / 2) {",
    "    __syncthreads();\n    tB += clock64() - tq; tq = clock64();\n    if (sm.nmap > LAT_MAP / 2) {")
rep("        sm.off[(int)threadIdx.x] = ex;\n        __syncthreads();",
    "        sm.off[(int)threadIdx.x] = ex;\n        __syncthreads();\n        tC += clock64() - tq; tq = clock64();")
rep("        __syncthreads();  // the tile's smem is reused by the next tile\n",
    "        __syncthreads();  // the tile's smem is reused by the next tile\n        tD += clock64() - tq; tq = clock64();\n")
rep("    cl.sync();  // the layer's arcs are out; beta of layer f-1 final in every rank\n",
    "    tq = clock64();\n    cl.sync();\n    tE += clock64() - tq;\n")
rep("  if (threadIdx.x == 0) {\n    CtwLatEntry& Ex = *sm.E;",
    "  if (threadIdx.x == 0) {\n    atomicAdd(&g_latprof[0], (unsigned long long)tA);\n"
    "    atomicAdd(&g_latprof[1], (unsigned long long)tB);\n    atomicAdd(&g_latprof[2], (unsigned long long)tC);\n"
    "    atomicAdd(&g_latprof[3], (unsigned long long)tD);\n    atomicAdd(&g_latprof[4], (unsigned long long)tE);\n"
    "    atomicAdd(&g_latprof[5], 1ULL);\n  }\n  if (threadIdx.x == 0) {\n    CtwLatEntry& Ex = *sm.E;")
S = S[:i0] + s + S[i1:]
S += """
extern "C" int ctw_latprof(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_latprof, sizeof(g_latprof));
  unsigned long long z[8] = {0};
  return (int)cudaMemcpyToSymbol(g_latprof, z, sizeof(z));
}
"""
p.write_text(S)
