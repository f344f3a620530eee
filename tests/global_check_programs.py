"""Programs for RunOptions::globalRaceCheck (builder-
defined, so the expectations are stated by construction rather than taken
from the reference, which has no global-race semantics): name -> (source,
expected global-race lines in report order).  With the option off, every
program must give the reference's own RunResult (goldens from
tests/make_edge_golden.py style runs in tests/golden/global_check.json)."""

def _host(kernel_launch, n=64):
    return (
        "int main(void) {\n"
        "  int* g;\n"
        f"  cudaMalloc(&g, {n} * sizeof(int));\n"
        f"  cudaMemset(g, 0, {n} * sizeof(int));\n"
        f"  {kernel_launch}\n"
        "  cudaDeviceSynchronize();\n"
        "  return 0;\n"
        "}\n")


PROGRAMS = {
    # disjoint per-thread slots: no cross-block conflict
    "disjoint": ("__global__ void k(int* g) {\n"
                 "  g[blockIdx.x * blockDim.x + threadIdx.x] = 1;\n"
                 "}\n" + _host("k<<<4, 16>>>(g);"), []),
    # every block writes the same word (line 2)
    "all_write_one": ("__global__ void k(int* g) {\n"
                      "  g[0] = blockIdx.x;\n"
                      "}\n" + _host("k<<<4, 1>>>(g);"), [2]),
    # thread 0 of every block increments g[0]: read and write on line 3
    "increment": ("__global__ void k(int* g) {\n"
                  "  if (threadIdx.x == 0) {\n"
                  "    g[0] += 1;\n"
                  "  }\n"
                  "}\n" + _host("k<<<3, 8>>>(g);"), [3]),
    # conflicts inside one block only: not a cross-block race
    "same_block": ("__global__ void k(int* g) {\n"
                   "  g[0] = threadIdx.x;\n"
                   "}\n" + _host("k<<<1, 32>>>(g);"), []),
    # block 1 reads (line 3) what block 0 writes (line 5) later on:
    # the read happens in an earlier sweep, so the write is the racing access
    "read_then_write": ("__global__ void k(int* g) {\n"
                        "  int x;\n"
                        "  if (blockIdx.x == 1) { x = g[5]; g[6] = x; }\n"
                        "  if (blockIdx.x == 0) {\n"
                        "    x = 1; x = x + 1; x = x + 1; x = x + 1; g[5] = x;\n"
                        "  }\n"
                        "}\n" + _host("k<<<2, 1>>>(g);"), [5]),
    # two grids, one after the other, on the same word: no race within a grid
    "two_grids": ("__global__ void k(int* g) {\n"
                  "  g[0] = blockIdx.x;\n"
                  "}\n"
                  "int main(void) {\n"
                  "  int* g;\n"
                  "  cudaMalloc(&g, 4 * sizeof(int));\n"
                  "  k<<<1, 1>>>(g);\n"
                  "  cudaDeviceSynchronize();\n"
                  "  k<<<1, 1>>>(g);\n"
                  "  cudaDeviceSynchronize();\n"
                  "  return 0;\n"
                  "}\n", []),
}
