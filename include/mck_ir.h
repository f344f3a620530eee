/*
 * mck_ir.h -- the step-exact kernel IR shared by the host compiler
 * (paper_1211_6193_b200/host/lower.cpp), the host-thread interpreter
 * (host/machine.cpp) and the sm_100a thread-stepping interpreter K1
 * (csrc/interp.cu).
 *
 * One IR instruction == one small step of the reference's continuation
 * machine (Machine::execThreadStep, /root/reference/proj/src/machine.cpp:493-1178:
 * every Item pop is one step, including no-op pops).  The expansion rules
 * are SURVEY.md Appendix B2; e.g. `a = b` is EXPR(1) + E(a) + RV(b) + STORE(1),
 * a `for` loop is SCOPE_PUSH + init + RV(c) + FORJUDGE + body + RV(n) +
 * POPVALUE + JMP + ... + SCOPE_POP.  OP_JMP is the only zero-step opcode: the
 * interpreters chase jumps inside the step that precedes them.
 *
 * Plain C, no torch types: included by C++ host code and by CUDA kernels.
 */
#ifndef MCK_IR_H
#define MCK_IR_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- C types, packed in one byte: base | ptr << 3 | array << 7 ----
 * (CType, ast.hpp:24-60; arrays are 1-D, the length lives in the symbol
 * tables because no run-time rule needs it). */
enum { MCK_VOID = 0, MCK_CHAR = 1, MCK_INT = 2, MCK_UINT = 3, MCK_LONG = 4, MCK_FLOAT = 5,
       MCK_DOUBLE = 6 };
#define MCK_T(base, ptr, arr) ((uint8_t)((base) | ((ptr) << 3) | ((arr) ? 0x80 : 0)))
#define MCK_T_BASE(t) ((t) & 7)
#define MCK_T_PTR(t) (((t) >> 3) & 15)
#define MCK_T_ARR(t) (((t) >> 7) & 1)
#define MCK_T_INT MCK_T(MCK_INT, 0, 0)
#define MCK_T_LONG MCK_T(MCK_LONG, 0, 0)
#define MCK_T_VOIDP MCK_T(MCK_VOID, 1, 0)

/* ---- value kinds (value.hpp:20) ---- */
enum { MCK_K_VOID = 0, MCK_K_INT = 1, MCK_K_FLOAT = 2, MCK_K_PTR = 3, MCK_K_STR = 4, MCK_K_LV = 5 };

/* ---- operators (ast.hpp:62-63) ---- */
enum { MCK_NEG = 0, MCK_NOT = 1, MCK_BITNOT = 2 };
enum { MCK_ADD, MCK_SUB, MCK_MUL, MCK_DIV, MCK_REM, MCK_SHL, MCK_SHR, MCK_LT, MCK_LE, MCK_GT,
       MCK_GE, MCK_EQ, MCK_NE, MCK_BAND, MCK_BXOR, MCK_BOR, MCK_LAND, MCK_LOR };
/* builtins (ast.hpp:89) */
enum { MCK_B_TID = 0, MCK_B_BID = 1, MCK_B_BDIM = 2, MCK_B_GDIM = 3, MCK_B_WARP = 4 };
/* __syncthreads variants (ast.hpp:96) */
enum { MCK_SYNC_PLAIN = 0, MCK_SYNC_AND = 1, MCK_SYNC_OR = 2, MCK_SYNC_COUNT = 3 };

/* ---- opcodes ---- */
enum {
  OP_NOP = 0,      /* no-op pop: Stmt(If/While/ExprSt/Decl/Empty), Expr expansion, last DeclStep */
  OP_SCOPE_PUSH,   /* Stmt(Block) / Stmt(For): push a scope                                 */
  OP_SCOPE_POP,    /* PopScope: owned objects die                                            */
  OP_JMP,          /* a = target; ZERO steps                                                  */
  OP_PUSH_INT,     /* t = type; value = (uint32)a | (int64)b << 32                            */
  OP_PUSH_FLT,     /* t = type; bits = (uint32)a | (uint64)b << 32                            */
  OP_PUSH_LOCAL,   /* t = declared type; a = frame slot                                       */
  OP_PUSH_GLOBAL,  /* t = type; a = global index                                              */
  OP_PUSH_BUILTIN, /* f = builtin var; a = component                                          */
  OP_UB,           /* a = MCK_UB_* code, b = name id: halting UB with a fixed message         */
  OP_LOADRV,       /* pop LValue, read (arrays decay), push value                             */
  OP_LOADKEEP,     /* pop LValue, read, push LValue + value                                   */
  OP_STORE,        /* StoreAssign                                                             */
  OP_STORE_OP,     /* StoreCompound, f = binop                                                */
  OP_STORE_INC,    /* StoreIncDec, a = delta, f = prefix                                      */
  OP_ADDROF,
  OP_DEREF,
  OP_INDEX,
  OP_UNARY,        /* f = MCK_NEG/NOT/BITNOT                                                  */
  OP_BINARY,       /* f = binop                                                               */
  OP_LOGRHS,       /* f = 1 for &&; a = target past the BOOLIFY when short-circuited          */
  OP_BOOLIFY,
  OP_TERNSEL,      /* a = else-branch target                                                  */
  OP_CAST,         /* t = cast type                                                           */
  OP_IFJUDGE,      /* a = target when false                                                   */
  OP_WHILEJUDGE,   /* a = loop exit                                                           */
  OP_FORJUDGE,     /* f = has condition; a = loop exit (the for's SCOPE_POP)                  */
  OP_POPVALUE,
  OP_RETURN,       /* ReturnUnwind; f = has value                                             */
  OP_BREAK,        /* a = target, b = scopes to pop                                           */
  OP_CONTINUE,     /* a = target, b = scopes to pop                                           */
  OP_CALL,         /* Invoke of a user function: a = function index, b = nargs              */
  OP_FALLOFF,      /* CallFrame popped by falling off the body                               */
  OP_SYNC,         /* Invoke(Sync): f = MCK_SYNC_*                                            */
  OP_DECL,         /* DeclStep: a = frame slot, b = local-table index, f = 1 dyn. shared      */
  OP_INITSTORE,    /* a = frame slot, t = declared type                                       */
  OP_PRINTF,       /* host only: a = string id, b = nargs                                     */
  OP_API,          /* host only: a = MCK_API_*, b = nargs                                     */
  OP_LAUNCH,       /* host only: a = kernel function index, b = nargs, f = 1 shmem | 2 stream */
  OP_COUNT
};

/* Halting UB with a fixed message (machine.cpp:666-1104). */
enum {
  MCK_UB_STRLIT = 1,     /* string literal in an unsupported position           */
  MCK_UB_MEMBER = 2,     /* unexpected member access                             */
  MCK_UB_UNBOUND = 3,    /* variable '<x>' is not bound in this scope (b = name) */
  MCK_UB_NOVALUE = 4,    /* cannot evaluate '<x>' as a value (b = name)          */
  MCK_UB_NOCALL = 5,     /* call of an unsupported function                      */
  MCK_UB_HOSTBUILTIN = 6 /* device builtin '<x>' referenced from host code       */
};

typedef struct mck_ins {
  uint8_t op;
  uint8_t t;
  uint8_t f;
  uint8_t pad;
  int32_t a;
  int32_t b;
  int32_t line;
} mck_ins;

/* A function: entry pc, frame slots (params first), return type. */
typedef struct mck_fn {
  int32_t entry;      /* pc of the body's first instruction                     */
  int32_t n_slots;    /* frame slots: params, then every declarator            */
  int32_t n_params;
  int32_t local_base; /* index of slot 0 in the local table                    */
  uint8_t ret;        /* return type                                            */
  uint8_t space;      /* 0 host, 1 device, 2 host+device, 3 kernel              */
  uint16_t pad;
  int32_t dyn_shared_slot; /* slot bound to the extern __shared__ array, or -1 */
} mck_fn;

/* One frame slot (param or declarator). */
typedef struct mck_local {
  int32_t size;   /* byte size of the object (arrays included) */
  int32_t name;   /* string id of the name                      */
  uint8_t type;
  uint8_t is_param;
  uint8_t is_dyn_shared;
  uint8_t pad;
} mck_local;

/* Device-global object as seen by K1 (cudaMalloc'ed or a __device__ global). */
typedef struct mck_gobj {
  uint32_t id;      /* reference object id                                   */
  uint32_t live;
  int64_t size;
  uint64_t base;    /* byte offset in the device arena                        */
  int32_t name;     /* string id                                              */
  int32_t pad;
} mck_gobj;

/* Runtime API ids (program.hpp:14-37). */
enum {
  MCK_API_MALLOC, MCK_API_FREE, MCK_API_MEMCPY, MCK_API_MEMCPY_ASYNC, MCK_API_MEMSET,
  MCK_API_DEVICE_SYNC, MCK_API_STREAM_CREATE, MCK_API_STREAM_DESTROY, MCK_API_STREAM_SYNC,
  MCK_API_STREAM_QUERY, MCK_API_STREAM_WAIT_EVENT, MCK_API_EVENT_CREATE, MCK_API_EVENT_DESTROY,
  MCK_API_EVENT_RECORD, MCK_API_EVENT_SYNC, MCK_API_EVENT_QUERY, MCK_API_EVENT_ELAPSED,
  MCK_API_GET_LAST_ERROR, MCK_API_GET_ERROR_STRING, MCK_API_DEVICE_GET_ATTR,
  MCK_API_DRIVER_VERSION, MCK_API_RUNTIME_VERSION, MCK_API_COUNT
};

/* ---- diagnostic templates emitted by K1 ----
 * A device diagnostic record carries the template id, the line, and up to
 * three integer parameters; the host formats it (machine.cpp:41-50 dedup). */
enum {
  MCK_D_RACE = 1,          /* Possible race on shared device memory detected at F:L.          */
  MCK_D_MEMBOUNDARY,       /* p0 = write?, p1 = target space (0 host, 1 global, 2 shared),
                              p2 = target (gid << 32 | bid) for shared                        */
  MCK_D_NULL_RW,           /* p0 = write?                                                      */
  MCK_D_DEAD,              /* p0 = write?, name                                                */
  MCK_D_OOB,               /* p0 = write?, p1 = len, p2 = offset, p3 = size, name              */
  MCK_D_UNINIT,            /* name                                                             */
  MCK_D_UNINIT_PTR,        /* name                                                             */
  MCK_D_NONPTR_AS_PTR,
  MCK_D_OVERFLOW,
  MCK_D_DIV0,
  MCK_D_REM0,
  MCK_D_SHIFT,
  MCK_D_PTR_ORDER_INT,     /* ordered comparison between a pointer and an integer             */
  MCK_D_PTR_ORDER_OBJ,     /* ordered comparison of pointers into different memory objects   */
  MCK_D_PTR_ADD,           /* invalid pointer addition                                         */
  MCK_D_PTR_SUB_OBJ,       /* subtraction of pointers into different memory objects           */
  MCK_D_PTR_SUB_VOID,      /* pointer subtraction on void pointers                             */
  MCK_D_PTR_OPERAND,       /* invalid pointer arithmetic operand                               */
  MCK_D_INT_MINUS_PTR,     /* integer minus pointer is not valid                               */
  MCK_D_VOID_ARITH,        /* arithmetic on void pointers                                      */
  MCK_D_PTR_OP,            /* invalid operation on pointer values                              */
  MCK_D_FLOAT_OP,          /* invalid operator on floating values                              */
  MCK_D_OPERANDS,          /* invalid operands                                                 */
  MCK_D_CONV_TO_PTR,       /* invalid conversion of a non-pointer value to a pointer          */
  MCK_D_CONV_TO_FLOAT,     /* invalid conversion to a floating type                            */
  MCK_D_FLOAT_RANGE,       /* floating value out of range in integer conversion               */
  MCK_D_PTR_TO_INT,        /* conversion of a pointer to an integer is not supported          */
  MCK_D_CONV,              /* invalid conversion                                               */
  MCK_D_DEREF_NONPTR,      /* dereference of a non-pointer value                               */
  MCK_D_SUBSCRIPT,         /* invalid subscript                                                */
  MCK_D_MODIFY_ARRAY,      /* cannot modify an array                                           */
  MCK_D_NEG_NONARITH,      /* negation of a non-arithmetic value                               */
  MCK_D_BITNOT_NONINT,     /* bitwise complement of a non-integer value                        */
  MCK_D_FIXED_UB,          /* OP_UB: p0 = MCK_UB_* code, name                                  */
  MCK_D_GRACE,             /* RunOptions::globalRaceCheck (builder-defined):
                              Possible race on global device memory detected at F:L.           */
  MCK_D_COUNT
};

#ifdef __cplusplus
}
#endif
#endif /* MCK_IR_H */
