"""CUDA-C programs for parity fixtures (test infrastructure).

* Fig. 1 (the reference corpus sum.cu, tests/golden/sum.cu) and its two
  mutants that keep line numbers;
* the scaled Fig. 1 reduction (SURVEY Appendix D gen.sh: one launch, host sum)
  and its racy variant without the second barrier (C2 shape);
* the barrier-divergence kernel of C4 (`if (v % 2) __syncthreads();`);
* random racy kernels (SURVEY Appendix D gen_rand.py shape): 3-11 statements
  over int / char / misaligned shared accesses, +=, tid-dependent loops,
  divergent stores and barriers; launched <<<{1,2,3}, {1,2,3,5,8,13,32,33}, 4*{4,8,16,64}>>>.
"""
import os
import random

HERE = os.path.dirname(os.path.abspath(__file__))


def fig1():
    with open(os.path.join(HERE, "golden", "sum.cu")) as f:
        return f.read()


def fig1_race():
    lines = fig1().split("\n")
    lines[13] = ""  # line 14: the second __syncthreads()
    return "\n".join(lines)


def fig1_deadlock():
    lines = fig1().split("\n")
    lines[11] = lines[11] + " __syncthreads();"  # inside `if (tid < bdim/2)`
    return "\n".join(lines)


def scaled(n, nthreads, racy=False):
    """Fig. 1 kernel verbatim (second barrier dropped when racy), host sum."""
    nb = n // nthreads
    sync2 = "" if racy else "  __syncthreads();"
    return f"""#include <stdio.h>
#include <cuda.h>
#define N {n}
#define NBLOCKS {nb}
#define NTHREADS (N/NBLOCKS)
__global__ void sum(int* in, int* out) {{
  extern __shared__ int shared[];
  int i, tid = threadIdx.x, bid = blockIdx.x, bdim = blockDim.x;
  shared[tid] = in[bid * bdim + tid];
  __syncthreads();
  if (tid < bdim/2) {{
    shared[tid] += shared[bdim/2 + tid];
  }}
{sync2}
  if (tid == 0) {{
    for (i=1; i != (bdim/2)+(bdim%2); ++i) {{
      shared[0] += shared[i];
    }}
    out[bid] = shared[0];
  }}
}}
int main(void) {{
  int i, s, *dev_in, *dev_out, host[N], part[NBLOCKS];
  for(i = 0; i != N; ++i) {{
    host[i] = (21*i + 29) % 100;
  }}
  cudaMalloc(&dev_in, N * sizeof(int));
  cudaMalloc(&dev_out, NBLOCKS * sizeof(int));
  cudaMemcpy(dev_in, host, N * sizeof(int), cudaMemcpyHostToDevice);
  sum<<<NBLOCKS, NTHREADS, NTHREADS * sizeof(int)>>>(dev_in, dev_out);
  cudaMemcpy(part, dev_out, NBLOCKS * sizeof(int), cudaMemcpyDeviceToHost);
  s = 0;
  for(i = 0; i != NBLOCKS; ++i) {{
    s += part[i];
  }}
  printf("OUTPUT: %d\\n", s);
  cudaFree(dev_in);
  cudaFree(dev_out);
  return 0;
}}
"""


def divergent_barrier(nblocks, nthreads, seed=0):
    """C4 miniature: per block all-even / all-odd / mixed values."""
    rng = random.Random(seed)
    vals = []
    for b in range(nblocks):
        pat = rng.randrange(3)
        for t in range(nthreads):
            v = rng.randrange(1 << 20)
            if pat == 0:
                v &= ~1
            elif pat == 1:
                v |= 1
            vals.append(v)
    n = nblocks * nthreads
    init = ", ".join(str(v) for v in vals)
    return f"""__global__ void k(int* in, int* out) {{
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  int v = in[g];
  if (v % 2) {{
    __syncthreads();
  }}
  out[g] = v;
}}
int main(void) {{
  int host[{n}] ;
  int i, *din, *dout;
  int vals[{n}] = {{{init}}};
  for (i = 0; i != {n}; ++i) host[i] = vals[i];
  cudaMalloc(&din, {n} * sizeof(int));
  cudaMalloc(&dout, {n} * sizeof(int));
  cudaMemcpy(din, host, {n} * sizeof(int), cudaMemcpyHostToDevice);
  k<<<{nblocks}, {nthreads}>>>(din, dout);
  cudaDeviceSynchronize();
  return 0;
}}
""", vals


def divergent_barrier_gen(nblocks, nthreads, seed=0):
    """Same kernel, inputs computed on the host by a formula (no initializer list)."""
    a = 2 * seed + 3
    return f"""__global__ void k(int* in, int* out) {{
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  int v = in[g];
  if (v % 2) {{
    __syncthreads();
  }}
  out[g] = v;
}}
int main(void) {{
  int host[{nblocks * nthreads}];
  int i, b, *din, *dout;
  for (i = 0; i != {nblocks * nthreads}; ++i) {{
    b = i / {nthreads};
    if (b % 3 == 0) host[i] = 2 * i;
    else if (b % 3 == 1) host[i] = 2 * i + 1;
    else host[i] = (i * {a} + b) % 7;
  }}
  cudaMalloc(&din, {nblocks * nthreads} * sizeof(int));
  cudaMalloc(&dout, {nblocks * nthreads} * sizeof(int));
  cudaMemcpy(din, host, {nblocks * nthreads} * sizeof(int), cudaMemcpyHostToDevice);
  k<<<{nblocks}, {nthreads}>>>(din, dout);
  cudaDeviceSynchronize();
  return 0;
}}
"""


def random_kernel(seed):
    rng = random.Random(seed)
    nb = rng.choice([1, 2, 3])
    nt = rng.choice([1, 2, 3, 5, 8, 13, 32, 33])
    sh = 4 * rng.choice([4, 8, 16, 64])
    m = sh // 4
    stmts = []
    for _ in range(rng.randint(3, 11)):
        k = rng.randrange(0, 7)
        c = rng.randrange(0, 5)
        r = rng.randrange(10)
        if r == 0:
            stmts.append(f"s[(t + {k}) % {m}] = t + {c};")
        elif r == 1:
            stmts.append(f"x += s[(t * {k + 1} + {c}) % {m}];")
        elif r == 2:
            stmts.append(f"c[(t + {k}) % {sh}] = t;")
        elif r == 3:
            stmts.append(f"x += c[(t * {k + 1} + {c}) % {sh}];")
        elif r == 4:
            stmts.append(f"*(int*)(c + ((t + {k}) % {sh - 4})) = x;")
        elif r == 5:
            stmts.append(f"x += *(int*)(c + ((t * {k + 1}) % {sh - 4}));")
        elif r == 6:
            stmts.append(f"s[(t + {k}) % {m}] += {c};")
        elif r == 7:
            stmts.append(f"for (j = 0; j < t % 3; ++j) {{ s[(t + j + {k}) % {m}] += j; }}")
        elif r == 8:
            stmts.append(f"if (t % 2 == 0) {{ s[(t + {k}) % {m}] = x; }}")
        else:
            stmts.append("__syncthreads();")
    body = "\n  ".join(stmts)
    src = f"""__global__ void k(int* g) {{
  extern __shared__ int s[];
  char* c;
  int t, j, x;
  c = (char*)s;
  t = threadIdx.x;
  x = 0;
  j = 0;
  {body}
  g[blockIdx.x * blockDim.x + t] = x + j;
}}
int main(void) {{
  int* g;
  cudaMalloc(&g, 4096);
  cudaMemset(g, 0, 4096);
  k<<<{nb}, {nt}, {sh}>>>(g);
  cudaDeviceSynchronize();
  return 0;
}}
"""
    return src


def random_kernel2(seed):
    """Richer random device programs (test infrastructure): device functions
    (with recursion), __syncthreads_and/or/count, local arrays and pointer
    arithmetic, intra-block global-memory conflicts, UB that halts a thread,
    two launches on two streams and a host that prints the results.
    Cross-BLOCK global conflicts are avoided (the B200 engine does not order
    different blocks inside a sweep; SURVEY Appendix E covers them)."""
    rng = random.Random(10_000 + seed)
    nb = rng.choice([1, 2, 3])
    nt = rng.choice([1, 2, 4, 7, 16, 32, 33, 48])
    sh = 4 * rng.choice([8, 16, 64])
    m = sh // 4
    body = []
    for _ in range(rng.randint(4, 12)):
        r = rng.randrange(16)
        k = rng.randrange(1, 7)
        if r == 0:
            body.append(f"s[(t * {k}) % {m}] = f(t + {k}, {rng.randrange(4)});")
        elif r == 1:
            body.append(f"x += s[(t + {k}) % {m}] * {rng.randrange(1, 4)};")
        elif r == 2:
            body.append(f"x += __syncthreads_count(t % {k} == 0);")
        elif r == 3:
            body.append(f"x += __syncthreads_or(x > {rng.randrange(20)}) + 2 * __syncthreads_and(t < {rng.randrange(1, 40)});")
        elif r == 4:
            body.append(f"loc[t % 4] = x; p = loc + (t % 3); x += *p + p[1];")
        elif r == 5:
            body.append(f"g[b * 64 + (t % 64)] += x;")  # block-private global slice; intra-block conflicts
        elif r == 6:
            body.append(f"j = 0; while (j < t % {k + 1}) {{ if (j == {k}) break; x = x * 3 - j; j++; }}")
        elif r == 7:
            body.append(f"for (j = 0; j < {k}; ++j) {{ if (j % 2) continue; c[(t + j) % {sh}] = (char)(x + j); }}")
        elif r == 8:
            body.append(f"x = (t & 1) ? x + c[(t * 5) % {sh}] : x - {k};")
        elif r == 9:
            body.append(f"if (t == {rng.randrange(nt + 2)}) {{ x = x / (t - t); }}")  # UB halt in one thread
        elif r == 10:
            body.append(f"x += fact(t % 6);")
        elif r == 11:
            body.append(f"s[(t + 1) % {m}] = x; __syncthreads(); x += s[t % {m}];")
        elif r == 12:
            body.append(f"if (t % {k + 1} == 0) {{ __syncthreads(); }}")  # may deadlock
        elif r == 13:
            body.append(f"x = (x << {rng.randrange(3)}) ^ (x >> 1) | {k};")
        elif r == 14:
            body.append(f"y = (long)x * {rng.choice([3, 100000, 2147483647])}; x = (int)(y % 1000);")
        else:
            body.append(f"g[b * 64 + ((t + {k}) % 64)] = g[b * 64 + (t % 64)] + 1;")
    code = "\n  ".join(body)
    k2 = rng.choice([1, 2])
    return f"""#include <stdio.h>
__device__ int f(int a, int d) {{
  if (d <= 0) return a % 7;
  return f(a * 3 + 1, d - 1) - d;
}}
__device__ long fact(int n) {{
  if (n < 2) return 1;
  return n * fact(n - 1);
}}
__global__ void k(int* g) {{
  extern __shared__ int s[];
  char* c;
  int t, j, x, b, loc[4], *p;
  long y;
  c = (char*)s;
  t = threadIdx.x;
  b = blockIdx.x;
  x = t;
  j = 0;
  for (j = 0; j < {m}; ++j) {{ if (j % {nt if nt > 0 else 1} == t) s[j] = j; }}
  __syncthreads();
  {code}
  g[b * 64 + (t % 64)] = x;
}}
__global__ void k2(int* g, int* out) {{
  int t = threadIdx.x, i, acc = 0;
  for (i = 0; i < {k2}; ++i) {{
    acc += g[(t * 5 + i) % {nb * 64}];
  }}
  out[t] = acc;
}}
int main(void) {{
  int *g, *out, h[16], i;
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaMalloc(&g, {nb * 64} * sizeof(int));
  cudaMalloc(&out, 16 * sizeof(int));
  cudaMemset(g, 0, {nb * 64} * sizeof(int));
  k<<<{nb}, {nt}, {sh}>>>(g);
  cudaDeviceSynchronize();
  k2<<<1, 16, 0, st>>>(g, out);
  cudaMemcpyAsync(h, out, 16 * sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  for (i = 0; i < 16; ++i) printf("%d ", h[i]);
  printf("\\n");
  return 0;
}}
"""


def concurrency_program(seed):
    """Host/device concurrency: two or three kernels on
    different streams in flight at once, async copies, events, and host loops
    that poll cudaStreamQuery / cudaEventQuery -- their iteration counts depend
    on the exact round-robin timing of the grids against the host thread."""
    rng = random.Random(20_000 + seed)
    nb1, nt1 = rng.choice([1, 2]), rng.choice([1, 3, 8, 17])
    nb2, nt2 = rng.choice([1, 2, 3]), rng.choice([2, 5, 16])
    loops1, loops2 = rng.randint(1, 12), rng.randint(1, 8)
    poll = rng.choice(["stream", "event", "both"])
    use_sync = rng.random() < 0.5
    return f"""#include <stdio.h>
__global__ void busy(int* g, int n) {{
  int t = threadIdx.x + blockIdx.x * blockDim.x, i, acc = t;
  for (i = 0; i < n; ++i) {{ acc = acc * 3 + i; }}
  g[t] = acc % 1000;
}}
__global__ void other(int* g, int off) {{
  extern __shared__ int s[];
  int t = threadIdx.x;
  s[t] = t + off;
  __syncthreads();
  g[off + blockIdx.x * blockDim.x + t] = s[(t + 1) % blockDim.x];
}}
int main(void) {{
  int *g, h[128], i, polls = 0, epolls = 0;
  cudaStream_t s1, s2;
  cudaEvent_t e1;
  cudaStreamCreate(&s1);
  cudaStreamCreate(&s2);
  cudaEventCreate(&e1);
  cudaMalloc(&g, 128 * sizeof(int));
  cudaMemset(g, 0, 128 * sizeof(int));
  busy<<<{nb1}, {nt1}, 0, s1>>>(g, {loops1});
  cudaEventRecord(e1, s1);
  other<<<{nb2}, {nt2}, {nt2} * sizeof(int), s2>>>(g, 64);
  busy<<<1, 4, 0, s2>>>(g + 100, {loops2});
  {"while (cudaStreamQuery(s1) != cudaSuccess) { polls++; }" if poll in ("stream", "both") else ""}
  {"while (cudaEventQuery(e1) == cudaErrorNotReady) { epolls++; }" if poll in ("event", "both") else ""}
  {"cudaStreamSynchronize(s2);" if use_sync else "cudaDeviceSynchronize();"}
  cudaMemcpyAsync(h, g, 128 * sizeof(int), cudaMemcpyDeviceToHost, s1);
  cudaStreamSynchronize(s1);
  printf("polls=%d epolls=%d\\n", polls, epolls);
  for (i = 0; i < 128; i += 7) printf("%d ", h[i]);
  printf("\\n");
  return 0;
}}
"""


def numeric_program(seed):
    """Device-side numerics and memory model: float/double arithmetic and
    conversions, __device__ globals, __host__ __device__ helpers called from
    both sides, unsigned / char / long wrap-around, shifts, pointer casts,
    compound assignments, ternaries, loops with break/continue."""
    rng = random.Random(30_000 + seed)
    nt = rng.choice([1, 2, 5, 8, 32])
    ops = []
    for _ in range(rng.randint(5, 14)):
        r = rng.randrange(12)
        c = rng.randint(1, 9)
        if r == 0:
            ops.append(f"f = f * {c}.5f - (float)t;")
        elif r == 1:
            ops.append(f"d = d / ({c} + t) + f;")
        elif r == 2:
            ops.append(f"u = u * {rng.choice([3, 65537, 2654435761])}u + t; u ^= u >> {c};")
        elif r == 3:
            ops.append(f"ch = (char)(ch + {c * 37}); acc += ch;")
        elif r == 4:
            ops.append(f"acc += twice(t + {c}) + (int)mix(d, {c});")
        elif r == 5:
            ops.append(f"gcount += t; acc += gcount % {c + 1};")
        elif r == 6:
            ops.append(f"l = l * {rng.choice([1000003, 7, -5])} + acc; acc = (int)(l % 1000);")
        elif r == 7:
            ops.append(f"acc = acc > {c * 10} ? acc - (int)f : acc + (int)d;")
        elif r == 8:
            ops.append(f"for (i = 0; i < {c}; ++i) {{ if (i == t) continue; if (i > 6) break; acc += i << (t % 4); }}")
        elif r == 9:
            ops.append(f"cp = (char*)&acc; acc += cp[{c % 4}];")
        elif r == 10:
            ops.append(f"acc %= {c + 2}; acc -= {c}; acc *= -{c};")
        else:
            ops.append(f"f = (float)(int)d; d = (double)u / {c}.0;")
    body = "\n  ".join(ops)
    return f"""#include <stdio.h>
__device__ int gcount;
__host__ __device__ int twice(int x) {{ return x + x; }}
__device__ double mix(double a, int b) {{ return a * b - b; }}
__global__ void k(int* out, float* fo, double* dout) {{
  int t = threadIdx.x, acc = t, i;
  unsigned u = 7u;
  char ch = 'a', *cp;
  long l = 1;
  float f = 1.25f;
  double d = 0.5;
  {body}
  out[t] = acc;
  fo[t] = f;
  dout[t] = d;
}}
int main(void) {{
  int *o, h[32], i;
  float *fo, hf[32];
  double *dd, hd[32];
  cudaMalloc(&o, 32 * sizeof(int));
  cudaMalloc(&fo, 32 * sizeof(float));
  cudaMalloc(&dd, 32 * sizeof(double));
  k<<<1, {nt}>>>(o, fo, dd);
  cudaMemcpy(h, o, {nt} * sizeof(int), cudaMemcpyDeviceToHost);
  cudaMemcpy(hf, fo, {nt} * sizeof(float), cudaMemcpyDeviceToHost);
  cudaMemcpy(hd, dd, {nt} * sizeof(double), cudaMemcpyDeviceToHost);
  for (i = 0; i < {nt}; ++i) printf("%d %f %f %d\\n", h[i], hf[i], hd[i], twice(h[i]));
  return 0;
}}
"""
