// ast.hpp -- syntax tree of the CUDA-C subset accepted by the checker.
//
// The accepted language and the source position every node carries follow
// the reference frontend (/root/reference/proj/src/parser.cpp:29-742,
// lexer.cpp:382-533): positions matter because the checker reports
// "<file>:<line>" of the token that created an expression.
// Nodes live in arenas owned by Unit; lowering (lower.cpp) annotates them and
// emits the step-exact IR of include/mck_ir.h.
#pragma once
#include <cstdint>
#include <deque>
#include <memory>
#include <string>
#include <vector>

namespace mckb {

struct Pos {
  int line = 0;
  int col = 0;
};

// C type: base, pointer depth, 1-D array length (-1 = not an array, 0 = unsized).
struct Ty {
  int base = 2;  // MCK_INT
  int ptr = 0;
  int64_t arr = -1;
  bool isArray() const { return arr >= 0; }
  bool isVoid() const { return base == 0 && ptr == 0 && arr < 0; }
  bool isFloat() const { return ptr == 0 && arr < 0 && (base == 5 || base == 6); }
  int64_t scalar() const;
  int64_t bytes() const { return isArray() ? scalar() * arr : scalar(); }
  uint8_t code() const;
  bool operator==(const Ty& o) const { return base == o.base && ptr == o.ptr && arr == o.arr; }
};

enum class EK { Int, Flt, Str, Name, Un, Bin, Asg, IncDec, Cond, Call, Idx, Mem, Cast, Sizeof,
                Launch, Builtin };
enum class SK { Block, If, While, For, Ret, Brk, Cont, ExprS, Decl, Empty };
enum class Bind { None, Local, Global, Func, Enum };
enum class Callee { None, User, Printf, Api, Sync };

struct Expr {
  EK k = EK::Int;
  Pos pos;
  int64_t ival = 0;
  double fval = 0;
  std::string text;
  std::string sval;
  Ty lit;           // literal type / resolved local type
  int op = 0;       // unary / binary operator (MCK_* in mck_ir.h)
  bool compound = false;
  bool prefix = false;
  int delta = 0;
  Ty castTy;
  Expr* a = nullptr;
  Expr* b = nullptr;
  Expr* c = nullptr;
  std::vector<Expr*> args;
  Expr* grid = nullptr;
  Expr* block = nullptr;
  Expr* shmem = nullptr;
  Expr* stream = nullptr;
  // lowering annotations
  Bind bind = Bind::None;
  int index = -1;       // local slot / global index / function index
  int64_t cval = 0;     // enum constant
  int builtin = 0, comp = 0;
  Callee callee = Callee::None;
  int calleeIndex = -1;  // function index or api id
  int syncKind = 0;
  int strId = -1;
};

struct Declarator {
  std::string name;
  Ty ty;
  Expr* init = nullptr;
  Pos pos;
  bool dynShared = false;
  int slot = -1;
};

struct Stmt {
  SK k = SK::Empty;
  Pos pos;
  std::vector<Stmt*> body;
  Expr* cond = nullptr;
  Stmt* thenS = nullptr;
  Stmt* elseS = nullptr;
  Stmt* loop = nullptr;
  Stmt* init = nullptr;
  Expr* incr = nullptr;
  Expr* e = nullptr;
  std::vector<Declarator> decls;
  bool externShared = false;
};

struct Param {
  std::string name;
  Ty ty;
  Pos pos;
};

// 0 host, 1 device, 2 host+device, 3 kernel (mck_fn.space)
struct Function {
  std::string name;
  Ty ret;
  std::vector<Param> params;
  Stmt* body = nullptr;
  int space = 0;
  Pos pos;
  std::string dynSharedName;
};

struct GlobalDef {
  std::string name;
  Ty ty;
  Expr* init = nullptr;
  bool device = false;
  Pos pos;
  int64_t ival = 0;
  double fval = 0;
  bool hasInit = false;
};

struct Unit {
  std::string filename;
  std::deque<Expr> exprs;
  std::deque<Stmt> stmts;
  std::vector<Function> fns;
  std::vector<GlobalDef> globals;
  Expr* newE(EK k, Pos p) {
    exprs.emplace_back();
    exprs.back().k = k;
    exprs.back().pos = p;
    return &exprs.back();
  }
  Stmt* newS(SK k, Pos p) {
    stmts.emplace_back();
    stmts.back().k = k;
    stmts.back().pos = p;
    return &stmts.back();
  }
};

// Frontend failure (lex / parse / semantic); never a run-time finding.
struct FrontendFailure {
  std::string stage;
  Pos pos;
  std::string message;
};

std::shared_ptr<Unit> parseUnit(const std::string& source, const std::string& filename);

}  // namespace mckb
