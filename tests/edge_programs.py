"""Edge-case programs of the whole-program parity corpus (test infrastructure):
step limits crossed inside grids, at the exact total and on the host, and the
capacity cases the reference has no bound for (deep recursion, wide blocks
racing on large shared arrays).  Goldens: tests/make_edge_golden.py runs the
reference on each (name -> {fname, step_limit, src}) and commits
tests/golden/edge_programs.json."""

SPIN = r"""__global__ void k(int* g) {
  int i;
  for (i = 0; i != %(iters)d; ++i) { g[threadIdx.x] += 1; }
}
int main(void) {
  int* g;
  int h[%(threads)d];
  cudaMalloc(&g, %(threads)d * sizeof(int));
  cudaMemset(g, 0, %(threads)d * sizeof(int));
  printf("before\n");
  k<<<%(blocks)d, %(threads)d>>>(g);
  cudaDeviceSynchronize();
  cudaMemcpy(h, g, %(threads)d * sizeof(int), cudaMemcpyDeviceToHost);
  printf("after %%d\n", h[0]);
  return 0;
}
"""

TWO_GRIDS = r"""__global__ void k(int* g, int n) {
  int i;
  for (i = 0; i != n; ++i) { g[blockIdx.x * blockDim.x + threadIdx.x] += i; }
}
int main(void) {
  int* g;
  int h[64];
  cudaMalloc(&g, 64 * sizeof(int));
  cudaMemset(g, 0, 64 * sizeof(int));
  k<<<2, 32>>>(g, 3);
  cudaDeviceSynchronize();
  k<<<4, 16>>>(g, 2);
  cudaDeviceSynchronize();
  cudaMemcpy(h, g, 64 * sizeof(int), cudaMemcpyDeviceToHost);
  printf("%d %d\n", h[0], h[63]);
  return 0;
}
"""

HOST_LOOP = r"""int main(void) {
  int x = 0;
  while (1) { x = x + 1; }
  return x;
}
"""

DEVICE_LOOP = r"""__global__ void k(int* g) {
  while (1) { g[threadIdx.x] = 1; }
}
int main(void) {
  int* g;
  cudaMalloc(&g, 64 * sizeof(int));
  k<<<1, 64>>>(g);
  cudaDeviceSynchronize();
  return 0;
}
"""


RECURSION = r"""__device__ int depth(int n) {
  int local = n * 3;
  if (n == 0) { return 0; }
  return depth(n - 1) + (local %% 7);
}
__global__ void k(int* g, int n) {
  g[blockIdx.x * blockDim.x + threadIdx.x] = depth(n + threadIdx.x %% 3);
}
int main(void) {
  int* g;
  int h[8];
  cudaMalloc(&g, 8 * sizeof(int));
  k<<<2, 4>>>(g, %(n)d);
  cudaMemcpy(h, g, 8 * sizeof(int), cudaMemcpyDeviceToHost);
  printf("%%d %%d %%d\n", h[0], h[5], h[7]);
  return 0;
}
"""

WIDE_RACE = r"""__global__ void k(int* g) {
  extern __shared__ int s[];
  int i;
  for (i = 0; i != 4; ++i) {
    s[(threadIdx.x * 4 + i) %% %(words)d] = threadIdx.x;
  }
  s[(threadIdx.x * 7) %% %(words)d] += 1;
  g[threadIdx.x] = s[threadIdx.x];
}
int main(void) {
  int* g;
  cudaMalloc(&g, %(threads)d * sizeof(int));
  k<<<%(blocks)d, %(threads)d, %(words)d * sizeof(int)>>>(g);
  cudaDeviceSynchronize();
  return 0;
}
"""


def edge_cases():
    """name -> (fname, step_limit, source).  Limits marked 'T' are resolved
    against the program's unlimited total by the golden maker."""
    out = {
        "limit_spin_in_grid": ("spin.cu", 1000, SPIN % dict(iters=10, blocks=1, threads=256)),
        "limit_spin_multi_block": ("spin2.cu", 20000, SPIN % dict(iters=40, blocks=8, threads=128)),
        "limit_spin_not_hit": ("spin3.cu", 1_000_000, SPIN % dict(iters=10, blocks=1, threads=256)),
        "limit_host_loop": ("hl.cu", 5000, HOST_LOOP),
        "limit_device_loop": ("dl.cu", 100_000, DEVICE_LOOP),
        "limit_two_grids_first": ("tg.cu", 500, TWO_GRIDS),
        "limit_two_grids_second": ("tg.cu", 1500, TWO_GRIDS),
    }
    for d in (-1, 0, 1):
        out[f"limit_two_grids_total{d:+d}"] = ("tg.cu", ("T", d), TWO_GRIDS)
    # capacity cases the reference has no bound for
    out["recursion_depth_64"] = ("rec.cu", 50_000_000, RECURSION % dict(n=62))
    out["recursion_depth_20"] = ("rec.cu", 50_000_000, RECURSION % dict(n=20))
    out["wide_race_1024x16k"] = ("wide.cu", 200_000_000, WIDE_RACE % dict(words=4096, threads=1024, blocks=1))
    out["wide_race_2x512x8k"] = ("wide2.cu", 200_000_000, WIDE_RACE % dict(words=2048, threads=512, blocks=2))
    # serial tails of blocks over 256 threads (several simulated threads per
    # GPU thread): thread 0 sums the partials alone for thousands of sweeps
    import gen_programs as gp
    out["tail_512x3"] = ("t512.cu", 200_000_000, gp.scaled(512 * 3, 512))
    out["tail_1024x2_racy"] = ("t1024.cu", 200_000_000, gp.scaled(1024 * 2, 1024, racy=True))
    return out
