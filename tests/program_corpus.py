"""The whole-program parity corpus (test infrastructure).

Each entry is (name, filename, source).  The golden RunResults were produced
by the unmodified reference (oracle/_ref/libmckref.so, Machine::run under
--schedule roundrobin) with tests/make_golden.py and are committed in
tests/golden/programs.json, so the GPU box needs no reference build."""
import gen_programs as gp

RICH = 500
CONC = 100
NUMS = 150


def corpus():
    out = [
        ("fig1", "sum.cu", gp.fig1()),
        ("fig1_race", "sum_race.cu", gp.fig1_race()),
        ("fig1_deadlock", "dl.cu", gp.fig1_deadlock()),
        ("scaled_256x64", "s.cu", gp.scaled(256 * 4, 256)),
        ("scaled_racy_256x2", "r.cu", gp.scaled(512, 256, racy=True)),
        ("scaled_33x3", "s3.cu", gp.scaled(99, 33)),
        ("scaled_racy_9x4", "r4.cu", gp.scaled(36, 9, racy=True)),
        ("divbar_4x8", "dl4.cu", gp.divergent_barrier_gen(4, 8, 0)),
        ("divbar_6x33", "dl6.cu", gp.divergent_barrier_gen(6, 33, 1)),
        ("divbar_3x64", "dl3.cu", gp.divergent_barrier_gen(3, 64, 2)),
    ]
    for i in range(300):
        out.append((f"rand{i}", f"rand{i}.cu", gp.random_kernel(i)))
    for i in range(RICH):
        out.append((f"rich{i}", f"rich{i}.cu", gp.random_kernel2(i)))
    for i in range(CONC):
        out.append((f"conc{i}", f"conc{i}.cu", gp.concurrency_program(i)))
    for i in range(NUMS):
        out.append((f"num{i}", f"num{i}.cu", gp.numeric_program(i)))
    return out


KEYS = ("exit", "output", "steps", "diags", "stuck_reports", "report_text", "reported", "main_return")


def project(run):
    """The fields compared for parity (RunResult + RaceState::reported)."""
    return {k: run.get(k) for k in KEYS}


HOST_STEP_LIMIT = 200_000


def host_corpus():
    """Host-only programs: the IR and value semantics without a GPU."""
    import gen_host_programs as gh
    out = [(f"host{i}", f"h{i}.cu", gh.host_program(i)) for i in range(400)]
    out += [(name, name + ".cu", src) for name, src in sorted(gh.HANDWRITTEN.items())]
    return out


FRONTEND_CASES = {
    "no_main": "int f(void) { return 0; }\n",
    "bad_token": "int main(void) { int x = 3 @ 4; return 0; }\n",
    "undeclared": "int main(void) { return y; }\n",
    "static_shared": "__global__ void k(void) { __shared__ int s[4]; }\nint main(void) { return 0; }\n",
    "printf_device": "__global__ void k(void) { printf(\"x\"); }\nint main(void) { return 0; }\n",
    "kernel_call": "__global__ void k(void) { }\nint main(void) { k(); return 0; }\n",
    "sync_host": "int main(void) { __syncthreads(); return 0; }\n",
    "break_outside": "int main(void) { break; return 0; }\n",
    "macro_fn": "#define F(x) x\nint main(void) { return 0; }\n",
    "array_init": "int main(void) { int a[3] = 1; return 0; }\n",
    "multi_dim": "int main(void) { int a[3][3]; return 0; }\n",
    "void_var": "int main(void) { void x; return 0; }\n",
    "kernel_ret": "__global__ int k(void) { return 1; }\nint main(void) { return 0; }\n",
    "redecl": "int main(void) { int x; int x; return 0; }\n",
    "unknown_api": "int main(void) { cudaFooBar(); return 0; }\n",
    "threadidx_host": "int main(void) { return threadIdx.x; }\n",
}
