// core.cuh -- value model and C arithmetic of the checked interpreter, shared
// by the host-thread interpreter (host/machine.cpp, g++ via nvcc) and the
// sm_100a thread-stepping kernel K1 (csrc/interp.cu).
//
// Semantics restated from the reference (file:line in /root/reference/proj):
//   Value / Location ........ include/minicudak/value.hpp:14-85
//   wrapToType .............. src/machine.cpp:117-124
//   arithResultType ......... src/machine.cpp:104-115
//   convertValueImpl ........ src/machine.cpp:131-176
//   binaryOpImpl ............ src/machine.cpp:180-387
//   UnaryOp ................. src/machine.cpp:893-920
// Diagnostics are returned as MCK_D_* template ids (include/mck_ir.h) in
// emission order; the caller attaches the source line and decides halting.
#pragma once
#include <stdint.h>

#include "mck_ir.h"

#if defined(__CUDACC__)
#define MCK_HD __host__ __device__ __forceinline__
#else
#define MCK_HD inline
#endif

namespace mck_core {

// A run-time value: 16 bytes.  Int: i.  Float: i holds the double's bits
// (float-typed values keep double precision until converted, machine.cpp:270).
// Ptr / LValue: (obj, i = offset) -- the reference's symbolic Location.
struct Val {
  uint8_t kind;
  uint8_t type;
  uint16_t pad;
  uint32_t obj;
  int64_t i;
};

MCK_HD double as_f(const Val& v) {
  union { int64_t i; double d; } u;
  u.i = v.i;
  return u.d;
}
MCK_HD int64_t f_bits(double d) {
  union { int64_t i; double d; } u;
  u.d = d;
  return u.i;
}
MCK_HD Val mk(uint8_t kind, uint8_t type, uint32_t obj, int64_t i) {
  Val v;
  v.kind = kind;
  v.type = type;
  v.pad = 0;
  v.obj = obj;
  v.i = i;
  return v;
}
MCK_HD Val v_void() { return mk(MCK_K_VOID, MCK_T_INT, 0, 0); }  // Value{} has type int
MCK_HD Val v_int(int64_t x, uint8_t t) { return mk(MCK_K_INT, t, 0, x); }
MCK_HD Val v_int(int64_t x) { return mk(MCK_K_INT, MCK_T_INT, 0, x); }
MCK_HD Val v_flt(double d, uint8_t t) { return mk(MCK_K_FLOAT, t, 0, f_bits(d)); }
MCK_HD Val v_ptr(uint32_t obj, int64_t off, uint8_t t) { return mk(MCK_K_PTR, t, obj, off); }
MCK_HD Val v_lv(uint32_t obj, int64_t off, uint8_t t) { return mk(MCK_K_LV, t, obj, off); }

// ---- types ----
MCK_HD bool t_is_void(uint8_t t) { return MCK_T_BASE(t) == MCK_VOID && MCK_T_PTR(t) == 0 && !MCK_T_ARR(t); }
MCK_HD bool t_is_float(uint8_t t) {
  return MCK_T_PTR(t) == 0 && !MCK_T_ARR(t) &&
         (MCK_T_BASE(t) == MCK_FLOAT || MCK_T_BASE(t) == MCK_DOUBLE);
}
// CType::scalarSize (ast.cpp:18-30): pointer = 8, else by base
MCK_HD int64_t t_scalar(uint8_t t) {
  if (MCK_T_PTR(t) > 0) return 8;
  switch (MCK_T_BASE(t)) {
    case MCK_CHAR: return 1;
    case MCK_INT: case MCK_UINT: case MCK_FLOAT: return 4;
    case MCK_LONG: case MCK_DOUBLE: return 8;
    default: return 0;
  }
}
// CType::element: arrays lose the array mark, pointers one level
MCK_HD uint8_t t_elem(uint8_t t) {
  if (MCK_T_ARR(t)) return (uint8_t)(t & 0x7F);
  return (uint8_t)MCK_T(MCK_T_BASE(t), MCK_T_PTR(t) - 1, 0);
}
MCK_HD uint8_t t_decay(uint8_t t) {
  if (!MCK_T_ARR(t)) return t;
  return (uint8_t)MCK_T(MCK_T_BASE(t), MCK_T_PTR(t) + 1, 0);
}
MCK_HD uint8_t t_addr(uint8_t t) {  // AddrOf result type (machine.cpp:862-864)
  uint8_t e = MCK_T_ARR(t) ? t_elem(t) : t;
  return (uint8_t)MCK_T(MCK_T_BASE(e), MCK_T_PTR(e) + 1, 0);
}

MCK_HD int64_t wrap_to(int64_t v, int base) {
  switch (base) {
    case MCK_CHAR: return (int8_t)v;
    case MCK_INT: return (int32_t)v;
    case MCK_UINT: return (int64_t)(uint32_t)v;
    default: return v;
  }
}

MCK_HD uint8_t arith_type(uint8_t l, uint8_t r) {
  int lb = MCK_T_BASE(l), rb = MCK_T_BASE(r);
  if (lb == MCK_DOUBLE || rb == MCK_DOUBLE) return MCK_T(MCK_DOUBLE, 0, 0);
  if (lb == MCK_FLOAT || rb == MCK_FLOAT) return MCK_T(MCK_FLOAT, 0, 0);
  if (lb == MCK_LONG || rb == MCK_LONG) return MCK_T_LONG;
  if (lb == MCK_UINT || rb == MCK_UINT) return MCK_T(MCK_UINT, 0, 0);
  return MCK_T_INT;
}

MCK_HD bool truthy(const Val& v) {
  switch (v.kind) {
    case MCK_K_INT: return v.i != 0;
    case MCK_K_FLOAT: return as_f(v) != 0.0;
    case MCK_K_PTR: return v.obj != 0;
    case MCK_K_STR: return true;
    default: return false;
  }
}

// Up to three diagnostics per step, in emission order.
struct Diags {
  uint8_t n;
  uint8_t code[3];
  MCK_HD void add(uint8_t c) {
    if (n < 3) code[n++] = c;
  }
};

// convertValueImpl.  Returns false when the thread halts.
MCK_HD bool convert(const Val& v, uint8_t t, Val& out, Diags& d) {
  if (t_is_void(t)) {
    out = v_void();
    return true;
  }
  if (MCK_T_PTR(t) > 0 && !MCK_T_ARR(t)) {
    if (v.kind == MCK_K_PTR) {
      out = v_ptr(v.obj, v.i, t);
      return true;
    }
    if (v.kind == MCK_K_INT && v.i == 0) {
      out = v_ptr(0, 0, t);
      return true;
    }
    d.add(MCK_D_CONV_TO_PTR);
    return false;
  }
  if (t_is_float(t)) {
    double x;
    if (v.kind == MCK_K_FLOAT)
      x = as_f(v);
    else if (v.kind == MCK_K_INT)
      x = (double)v.i;
    else {
      d.add(MCK_D_CONV_TO_FLOAT);
      return false;
    }
    if (MCK_T_BASE(t) == MCK_FLOAT) x = (double)(float)x;
    out = v_flt(x, t);
    return true;
  }
  if (v.kind == MCK_K_INT) {
    out = v_int(wrap_to(v.i, MCK_T_BASE(t)), t);
    return true;
  }
  if (v.kind == MCK_K_FLOAT) {
    double x = as_f(v);
    if (!(x >= -9.3e18 && x <= 9.3e18)) {
      d.add(MCK_D_FLOAT_RANGE);
      out = v_int(0, t);
      return true;
    }
    out = v_int(wrap_to((int64_t)x, MCK_T_BASE(t)), t);
    return true;
  }
  d.add(v.kind == MCK_K_PTR ? MCK_D_PTR_TO_INT : MCK_D_CONV);
  return false;
}

// __builtin_*_overflow on int64 (machine.cpp:296-319): wrapped result + flag
MCK_HD bool add_ovf(int64_t a, int64_t b, int64_t* r) {
  int64_t x = (int64_t)((uint64_t)a + (uint64_t)b);
  *r = x;
  return ((a ^ x) & (b ^ x)) < 0;
}
MCK_HD bool sub_ovf(int64_t a, int64_t b, int64_t* r) {
  int64_t x = (int64_t)((uint64_t)a - (uint64_t)b);
  *r = x;
  return ((a ^ b) & (a ^ x)) < 0;
}
MCK_HD bool mul_ovf(int64_t a, int64_t b, int64_t* r) {
  int64_t lo = (int64_t)((uint64_t)a * (uint64_t)b);
  *r = lo;
#if defined(__CUDA_ARCH__)
  int64_t hi = __mul64hi(a, b);
#else
  int64_t hi = (int64_t)(((__int128)a * (__int128)b) >> 64);
#endif
  return hi != (lo >> 63);
}

// binaryOpImpl.  Returns false when the thread halts.
MCK_HD bool binop(int op, const Val& l, const Val& r, Val& out, Diags& d) {
  if (l.kind == MCK_K_PTR || r.kind == MCK_K_PTR) {
    switch (op) {
      case MCK_EQ:
      case MCK_NE: {
        bool eq;
        if (l.kind == MCK_K_PTR && r.kind == MCK_K_PTR)
          eq = l.obj == r.obj && l.i == r.i;
        else if (l.kind == MCK_K_PTR)
          eq = r.kind == MCK_K_INT && r.i == 0 && l.obj == 0;
        else
          eq = l.kind == MCK_K_INT && l.i == 0 && r.obj == 0;
        out = v_int((op == MCK_EQ) == eq ? 1 : 0);
        return true;
      }
      case MCK_LT: case MCK_LE: case MCK_GT: case MCK_GE: {
        if (l.kind != MCK_K_PTR || r.kind != MCK_K_PTR) {
          d.add(MCK_D_PTR_ORDER_INT);
          return false;
        }
        if (l.obj != r.obj) d.add(MCK_D_PTR_ORDER_OBJ);
        int c = l.obj < r.obj ? -1 : l.obj > r.obj ? 1 : (l.i < r.i ? -1 : l.i > r.i ? 1 : 0);
        bool res = op == MCK_LT ? c < 0 : op == MCK_LE ? c <= 0 : op == MCK_GT ? c > 0 : c >= 0;
        out = v_int(res ? 1 : 0);
        return true;
      }
      case MCK_ADD:
      case MCK_SUB: {
        if (l.kind == MCK_K_PTR && r.kind == MCK_K_PTR) {
          if (op != MCK_SUB) { d.add(MCK_D_PTR_ADD); return false; }
          if (l.obj != r.obj) { d.add(MCK_D_PTR_SUB_OBJ); return false; }
          int64_t es = t_scalar(t_elem(l.type));
          if (es == 0) { d.add(MCK_D_PTR_SUB_VOID); return false; }
          out = v_int((l.i - r.i) / es, MCK_T_LONG);
          return true;
        }
        const Val& p = l.kind == MCK_K_PTR ? l : r;
        const Val& x = l.kind == MCK_K_PTR ? r : l;
        if (x.kind != MCK_K_INT) { d.add(MCK_D_PTR_OPERAND); return false; }
        if (op == MCK_SUB && l.kind != MCK_K_PTR) { d.add(MCK_D_INT_MINUS_PTR); return false; }
        int64_t es = t_scalar(t_elem(p.type));
        if (es == 0) { d.add(MCK_D_VOID_ARITH); return false; }
        int64_t delta = (int64_t)((uint64_t)x.i * (uint64_t)es);
        out = v_ptr(p.obj, op == MCK_ADD ? p.i + delta : p.i - delta, p.type);
        return true;
      }
      default:
        d.add(MCK_D_PTR_OP);
        return false;
    }
  }
  const uint8_t rt = arith_type(l.type, r.type);
  if (t_is_float(rt)) {
    if (op == MCK_REM || op == MCK_SHL || op == MCK_SHR || op == MCK_BAND || op == MCK_BOR ||
        op == MCK_BXOR) {
      d.add(MCK_D_FLOAT_OP);
      return false;
    }
    double a = l.kind == MCK_K_FLOAT ? as_f(l) : (double)l.i;
    double b = r.kind == MCK_K_FLOAT ? as_f(r) : (double)r.i;
    switch (op) {
      case MCK_ADD: out = v_flt(a + b, rt); return true;
      case MCK_SUB: out = v_flt(a - b, rt); return true;
      case MCK_MUL: out = v_flt(a * b, rt); return true;
      case MCK_DIV: out = v_flt(a / b, rt); return true;
      case MCK_LT: out = v_int(a < b); return true;
      case MCK_LE: out = v_int(a <= b); return true;
      case MCK_GT: out = v_int(a > b); return true;
      case MCK_GE: out = v_int(a >= b); return true;
      case MCK_EQ: out = v_int(a == b); return true;
      case MCK_NE: out = v_int(a != b); return true;
      default: return false;
    }
  }
  if (l.kind != MCK_K_INT || r.kind != MCK_K_INT) {
    d.add(MCK_D_OPERANDS);
    return false;
  }
  const int64_t a = l.i, b = r.i;
  const int base = MCK_T_BASE(rt);
  const bool uns = base == MCK_UINT;
  const int width = base == MCK_LONG ? 64 : 32;
  int64_t raw = 0;
  bool ovf = false, check = false;
  switch (op) {
    case MCK_ADD: ovf = add_ovf(a, b, &raw); check = !ovf; break;
    case MCK_SUB: ovf = sub_ovf(a, b, &raw); check = !ovf; break;
    case MCK_MUL: ovf = mul_ovf(a, b, &raw); check = !ovf; break;
    case MCK_DIV:
      if (b == 0) { d.add(MCK_D_DIV0); return false; }
      if (uns) { raw = (int64_t)((uint32_t)a / (uint32_t)b); break; }
      if (a == INT64_MIN && b == -1) { ovf = true; raw = a; break; }
      raw = a / b;
      check = true;
      break;
    case MCK_REM:
      if (b == 0) { d.add(MCK_D_REM0); return false; }
      if (uns) { raw = (int64_t)((uint32_t)a % (uint32_t)b); break; }
      if (a == INT64_MIN && b == -1) { raw = 0; break; }
      raw = a % b;
      check = true;
      break;
    case MCK_SHL:
    case MCK_SHR: {
      int64_t s = b;
      if (s < 0 || s >= width) {
        d.add(MCK_D_SHIFT);
        s &= width - 1;
      }
      uint64_t ua = uns ? (uint64_t)(uint32_t)a : (uint64_t)a;
      if (op == MCK_SHL)
        raw = (int64_t)(ua << s);
      else if (uns)
        raw = (int64_t)((uint32_t)a >> s);
      else
        raw = a >> s;
      break;
    }
    case MCK_LT: case MCK_LE: case MCK_GT: case MCK_GE: case MCK_EQ: case MCK_NE: {
      int64_t wa = wrap_to(a, base), wb = wrap_to(b, base);
      bool res = op == MCK_LT ? wa < wb : op == MCK_LE ? wa <= wb : op == MCK_GT ? wa > wb
               : op == MCK_GE ? wa >= wb : op == MCK_EQ ? wa == wb : wa != wb;
      out = v_int(res ? 1 : 0);
      return true;
    }
    case MCK_BAND: raw = a & b; break;
    case MCK_BOR: raw = a | b; break;
    case MCK_BXOR: raw = a ^ b; break;
    default: return false;
  }
  if (ovf && !uns) d.add(MCK_D_OVERFLOW);
  const int64_t w = wrap_to(raw, base);
  if (check && !uns && w != raw) d.add(MCK_D_OVERFLOW);
  out = v_int(w, rt);
  return true;
}

// UnaryOp (machine.cpp:893-920).  Returns false when the thread halts.
MCK_HD bool unop(int op, const Val& v, Val& out, Diags& d) {
  switch (op) {
    case MCK_NEG:
      if (v.kind == MCK_K_FLOAT) {
        out = v_flt(-as_f(v), v.type);
        return true;
      }
      if (v.kind == MCK_K_INT) return binop(MCK_SUB, v_int(0, v.type), v, out, d);
      d.add(MCK_D_NEG_NONARITH);
      return false;
    case MCK_NOT:
      out = v_int(truthy(v) ? 0 : 1);
      return true;
    default: {
      if (v.kind != MCK_K_INT) {
        d.add(MCK_D_BITNOT_NONINT);
        return false;
      }
      uint8_t rt = arith_type(v.type, MCK_T_INT);
      out = v_int(wrap_to(~v.i, MCK_T_BASE(rt)), rt);
      return true;
    }
  }
}

// Little-endian assembly of a scalar read (memory.cpp:172-181).
MCK_HD Val decode_scalar(uint64_t raw, uint8_t t) {
  int base = MCK_T_BASE(t);
  if (base == MCK_FLOAT) {
    union { uint32_t u; float f; } u;
    u.u = (uint32_t)raw;
    return v_flt((double)u.f, t);
  }
  if (base == MCK_DOUBLE) return mk(MCK_K_FLOAT, t, 0, (int64_t)raw);
  int64_t x;
  switch (base) {
    case MCK_CHAR: x = (int8_t)raw; break;
    case MCK_INT: x = (int32_t)raw; break;
    case MCK_UINT: x = (uint32_t)raw; break;
    default: x = (int64_t)raw; break;
  }
  return v_int(x, t);
}

// pokeValue raw encoding (memory.cpp:184-206).
MCK_HD uint64_t encode_scalar(const Val& v, uint8_t t) {
  if (v.kind == MCK_K_PTR) return ((uint64_t)v.obj << 32) | ((uint64_t)v.i & 0xffffffffu);
  if (MCK_T_PTR(t) > 0) return (uint64_t)v.i;
  if (MCK_T_BASE(t) == MCK_FLOAT) {
    union { uint32_t u; float f; } u;
    u.f = (float)as_f(v);
    return u.u;
  }
  if (MCK_T_BASE(t) == MCK_DOUBLE) return (uint64_t)v.i;
  return (uint64_t)v.i;
}

}  // namespace mck_core
