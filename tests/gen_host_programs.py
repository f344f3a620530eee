"""Random HOST-ONLY CUDA-C programs (test infrastructure).

They exercise the step-exact IR and the value semantics shared by the host
interpreter and the K1 kernel (core.cuh): C integer/floating arithmetic with
overflow / division / shift diagnostics, conversions, pointers and arrays,
pointer arithmetic and comparisons, calls with recursion, loops with break and
continue, ternaries, short-circuit logic, casts, printf conversions, sizeof,
uninitialised reads, out-of-bounds and dead-object accesses.  Golden results
come from the reference itself (tests/make_golden.py)."""
import random

TYPES = ["int", "char", "unsigned", "long", "float", "double"]


def _lit(rng, t):
    if t in ("float", "double"):
        return f"{rng.uniform(-100, 100):.3f}" + ("f" if t == "float" and rng.random() < 0.5 else "")
    choices = [0, 1, 2, 3, 7, -1, -5, 100, 127, 255, 65535, 2147483647, -2147483647]
    v = rng.choice(choices)
    if t == "unsigned":
        return f"{abs(v)}u"
    if t == "long" and rng.random() < 0.5:
        return f"{v}L"
    return str(v)


def host_program(seed):
    rng = random.Random(seed)
    vars_ = {}
    decls, body = [], []
    for i in range(rng.randint(3, 6)):
        t = rng.choice(TYPES)
        n = f"v{i}"
        vars_[n] = t
        decls.append(f"  {t} {n} = {_lit(rng, t)};")
    decls.append("  int a[8]; int k; int *p; char buf[6];")
    decls.append("  long acc = 0;")
    names = list(vars_)
    ops = ["+", "-", "*", "/", "%", "<<", ">>", "&", "|", "^", "<", "<=", "==", "!=", "&&", "||"]
    def expr(depth=0):
        r = rng.random()
        if depth > 2 or r < 0.3:
            return rng.choice(names + [_lit(rng, "int")])
        if r < 0.45:
            return f"({rng.choice(['-', '!', '~'])}{expr(depth + 1)})"
        if r < 0.55:
            return f"(({rng.choice(['int', 'char', 'long', 'unsigned', 'double'])}){expr(depth + 1)})"
        if r < 0.62:
            return f"({expr(depth + 1)} ? {expr(depth + 1)} : {expr(depth + 1)})"
        return f"({expr(depth + 1)} {rng.choice(ops)} {expr(depth + 1)})"
    for _ in range(rng.randint(4, 12)):
        r = rng.randrange(14)
        x = rng.choice(names)
        if r == 0:
            body.append(f"  {x} = {expr()};")
        elif r == 1:
            body.append(f"  {x} {rng.choice(['+=', '-=', '*=', '<<=', '|=', '^='])} {expr()};")
        elif r == 2:
            body.append(f"  for (k = 0; k < 8; ++k) {{ a[k] = k * {rng.randint(1, 9)} - {rng.randint(0, 20)}; }}")
        elif r == 3:
            body.append(f"  for (k = 0; k != 8; k++) {{ if (a[k] % 3 == 0) continue; acc += a[k]; if (acc > {rng.randint(5, 60)}) break; }}")
        elif r == 4:
            body.append(f"  p = a + {rng.randint(0, 7)}; acc += *p + p[{rng.randint(-1, 1)}] + (p - a);")
        elif r == 5:
            body.append(f"  printf(\"%d %u %c|\\n\", (int)({expr()}), (unsigned)({expr()}), 65 + (k & 7));")
        elif r == 6:
            body.append(f"  printf(\"%f %5.1f %s\\n\", (double){x}, (float){expr()}, cudaGetErrorString({rng.choice([0, 11, 17, 99])}));")
        elif r == 7:
            body.append(f"  acc += fib({rng.randint(0, 9)}) + sq({expr()});")
        elif r == 8:
            body.append(f"  k = 0; while (k < {rng.randint(0, 6)}) {{ acc = acc * 3 + k; k++; }}")
        elif r == 9:
            body.append(f"  {x}++; --{x}; acc += sizeof({x}) + sizeof(long) + sizeof(char*);")
        elif r == 10:
            body.append(f"  buf[{rng.randint(0, 5)}] = (char){expr()}; acc += buf[{rng.randint(0, 5)}];")
        elif r == 11:
            body.append(f"  acc += (p > a) + (p == a) + (p != 0);")
        elif r == 12:
            body.append(f"  acc = acc {rng.choice(['/', '%'])} ({x} % 4);")
        else:
            body.append(f"  acc += a[{rng.choice([0, 3, 7, 8, -1])}];")
    body.append("  printf(\"acc=%d\\n\", acc);")
    body.append(f"  return {rng.choice(['0', '(int)acc & 7', '3'])};")
    return ("#include <stdio.h>\n"
            "int fib(int n) { if (n < 2) return n; return fib(n - 1) + fib(n - 2); }\n"
            "long sq(long x) { return x * x; }\n"
            "int* dangle(void) { int z = 5; return &z; }\n"
            "int main(void) {\n" + "\n".join(decls) + "\n  p = a;\n" + "\n".join(body) + "\n}\n")


HANDWRITTEN = {
    "dead_pointer": """int* dangle(void) { int z = 5; return &z; }
int main(void) { int* q = dangle(); return *q; }
""",
    "null_deref": """int main(void) { int* q = 0; *q = 3; return 0; }
""",
    "uninit": """#include <stdio.h>
int main(void) { int x; int y = x + 1; printf("%d\\n", y > 0); return 0; }
""",
    "oob": """int main(void) { int a[4]; a[4] = 1; return 0; }
""",
    "api_errors": """#include <stdio.h>
int main(void) {
  int *d, h[4];
  cudaMalloc(&d, 16);
  printf("%d\\n", cudaMemcpy(h, d, 16, cudaMemcpyHostToDevice));
  printf("%d %d\\n", cudaGetLastError(), cudaGetLastError());
  cudaFree(d);
  printf("%d\\n", cudaFree(d));
  h[0] = 1;
  return h[0];
}
""",
    "memcpy_roundtrip": """#include <stdio.h>
int main(void) {
  int *d, h[4], g[4], i;
  for (i = 0; i < 4; ++i) h[i] = i * 7;
  cudaMalloc(&d, 16);
  cudaMemcpy(d, h, 16, cudaMemcpyHostToDevice);
  cudaMemset(d, 0, 4);
  cudaMemcpy(g, d, 16, cudaMemcpyDeviceToHost);
  printf("%d %d %d %d\\n", g[0], g[1], g[2], g[3]);
  return 0;
}
""",
    "host_touches_device": """int main(void) { int* d; cudaMalloc(&d, 8); d[0] = 1; return 0; }
""",
    "streams_events": """#include <stdio.h>
int main(void) {
  cudaStream_t s; cudaEvent_t e; float ms;
  cudaStreamCreate(&s);
  cudaEventCreate(&e);
  cudaEventRecord(e, s);
  printf("%d\\n", cudaEventQuery(e));
  cudaEventSynchronize(e);
  printf("%d\\n", cudaEventQuery(e));
  cudaEventElapsedTime(&ms, e, e);
  printf("%f %d\\n", ms, cudaStreamQuery(s));
  cudaStreamDestroy(s);
  cudaDeviceSynchronize();
  return 0;
}
""",
    "step_limit": """int main(void) { int i = 0; while (1) { i++; } return 0; }
""",
}
