"""Programs for the exhaustive-interleaving oracle (oracleRace,
oracle.cpp:73-154): name -> (source, options).  Goldens come from the
reference's own oracleRace (tests/make_oracle_golden.py)."""

K = r"""__global__ void k(int* g) {
  extern __shared__ int s[];
%(body)s
}
int main(void) {
  int* g;
  cudaMalloc(&g, 64 * sizeof(int));
  cudaMemset(g, 0, 64 * sizeof(int));
  k<<<%(grid)d, %(block)d, %(shmem)d>>>(g);
  cudaDeviceSynchronize();
  return 0;
}
"""


def prog(body, grid=1, block=2, shmem=16):
    return K % dict(body=body, grid=grid, block=block, shmem=shmem)


D = dict(max_interleavings=1_000_000, max_threads=3, max_accesses=8)

PROGRAMS = {
    "neighbour_race": (prog("  s[threadIdx.x] = threadIdx.x;\n  g[threadIdx.x] = s[(threadIdx.x + 1) % blockDim.x];"), D),
    "neighbour_synced": (prog("  s[threadIdx.x] = threadIdx.x;\n  __syncthreads();\n"
                              "  g[threadIdx.x] = s[(threadIdx.x + 1) % blockDim.x];"), D),
    "three_threads": (prog("  s[threadIdx.x] = threadIdx.x;\n  g[threadIdx.x] = s[(threadIdx.x + 1) % blockDim.x];",
                           block=3), D),
    "disjoint": (prog("  s[threadIdx.x] = 1;\n  s[threadIdx.x] += 2;"), D),
    "read_read": (prog("  g[threadIdx.x] = s[0] + s[1];"), D),
    "write_write": (prog("  s[0] = threadIdx.x;"), D),
    "conditional_race": (prog("  if (threadIdx.x == 0) { s[0] = 5; }\n  __syncthreads();\n"
                              "  if (s[0] == 5 && threadIdx.x == 1) { s[1] = 1; }\n"
                              "  if (threadIdx.x == 0) { g[0] = s[1]; }"), D),
    "value_dependent": (prog("  s[threadIdx.x] = threadIdx.x + 1;\n  if (s[1 - threadIdx.x] != 0) { g[threadIdx.x] = 7; }"), D),
    "sync_count": (prog("  s[threadIdx.x] = __syncthreads_count(threadIdx.x == 0);\n  __syncthreads();\n"
                        "  g[threadIdx.x] = s[0] + s[1];"), D),
    "two_blocks": (prog("  s[0] = blockIdx.x;\n  g[blockIdx.x] = s[0];", grid=2, block=1), D),
    "two_blocks_two_threads": (prog("  s[threadIdx.x] = blockIdx.x;\n  g[threadIdx.x] = s[1 - threadIdx.x];",
                                    grid=2, block=2), dict(D, max_threads=4)),
    "char_vs_int": (prog("  char* c = (char*)s;\n  if (threadIdx.x == 0) { s[0] = 0x01020304; }\n"
                         "  if (threadIdx.x == 1) { c[2] = 9; }"), D),
    "deadlock": (prog("  s[threadIdx.x] = 1;\n  if (threadIdx.x == 0) { __syncthreads(); }"), D),
    "loop": (prog("  int i;\n  for (i = 0; i != 2; ++i) { s[i] += threadIdx.x; }"), D),
    "four_threads": (prog("  s[threadIdx.x] = threadIdx.x;\n  __syncthreads();\n  g[threadIdx.x] = s[3 - threadIdx.x];",
                          block=4), dict(D, max_threads=4)),
    "budget": (prog("  s[threadIdx.x] = threadIdx.x;\n  g[threadIdx.x] = s[(threadIdx.x + 1) % blockDim.x];"),
               dict(D, max_interleavings=10)),
    "too_many_threads": (prog("  s[threadIdx.x] = 1;", block=4), D),
    "no_kernel": ("int main(void) { int x = 3; return x - 3; }\n", D),
}
