// lower.cpp -- name resolution, static checks and step-exact IR generation.
//
// Provenance: the name resolution and call / launch checks (resolveName,
// resolveCall, resolveLaunch) restate the reference's Lowerer closely, since
// their diagnostics must match it byte for byte; the IR emission (stmt / ex /
// rv) is this project's own design.
//
// Static rules follow the reference lowering (/root/reference/proj/src/lower.cpp:
// main checks 143-173, globals 175-207, call classification 467-535, launch
// 551-573, sizeof typing 576-640).  Code generation follows the continuation
// expansion of Machine::execThreadStep (src/machine.cpp:538-760) so that one IR
// instruction is exactly one small step; jumps are free.
#include <cstdio>
#include <map>
#include <optional>

#include "program.hpp"

namespace mckb {

int Program::intern(const std::string& s) {
  auto it = ids_.find(s);
  if (it != ids_.end()) return it->second;
  int id = static_cast<int>(strings.size());
  strings.push_back(s);
  ids_[s] = id;
  return id;
}

namespace {

[[noreturn]] void semErr(Pos p, const std::string& m) { throw FrontendFailure{"semantic", p, m}; }

struct ApiEntry { int id, mn, mx; };
const std::map<std::string, ApiEntry>& apis() {
  static const std::map<std::string, ApiEntry> m = {
      {"cudaMalloc", {MCK_API_MALLOC, 2, 2}}, {"cudaFree", {MCK_API_FREE, 1, 1}},
      {"cudaMemcpy", {MCK_API_MEMCPY, 4, 4}}, {"cudaMemcpyAsync", {MCK_API_MEMCPY_ASYNC, 4, 5}},
      {"cudaMemset", {MCK_API_MEMSET, 3, 3}}, {"cudaDeviceSynchronize", {MCK_API_DEVICE_SYNC, 0, 0}},
      {"cudaStreamCreate", {MCK_API_STREAM_CREATE, 1, 1}},
      {"cudaStreamDestroy", {MCK_API_STREAM_DESTROY, 1, 1}},
      {"cudaStreamSynchronize", {MCK_API_STREAM_SYNC, 1, 1}},
      {"cudaStreamQuery", {MCK_API_STREAM_QUERY, 1, 1}},
      {"cudaStreamWaitEvent", {MCK_API_STREAM_WAIT_EVENT, 2, 3}},
      {"cudaEventCreate", {MCK_API_EVENT_CREATE, 1, 1}},
      {"cudaEventDestroy", {MCK_API_EVENT_DESTROY, 1, 1}},
      {"cudaEventRecord", {MCK_API_EVENT_RECORD, 1, 2}},
      {"cudaEventSynchronize", {MCK_API_EVENT_SYNC, 1, 1}},
      {"cudaEventQuery", {MCK_API_EVENT_QUERY, 1, 1}},
      {"cudaEventElapsedTime", {MCK_API_EVENT_ELAPSED, 3, 3}},
      {"cudaGetLastError", {MCK_API_GET_LAST_ERROR, 0, 0}},
      {"cudaGetErrorString", {MCK_API_GET_ERROR_STRING, 1, 1}},
      {"cudaDeviceGetAttribute", {MCK_API_DEVICE_GET_ATTR, 2, 3}},
      {"cudaDriverGetVersion", {MCK_API_DRIVER_VERSION, 1, 1}},
      {"cudaRuntimeGetVersion", {MCK_API_RUNTIME_VERSION, 1, 1}}};
  return m;
}

const std::map<std::string, int64_t>& enumConsts() {
  static const std::map<std::string, int64_t> m = {
      {"cudaMemcpyHostToHost", 0}, {"cudaMemcpyHostToDevice", 1}, {"cudaMemcpyDeviceToHost", 2},
      {"cudaMemcpyDeviceToDevice", 3}, {"cudaSuccess", 0}, {"cudaErrorInvalidValue", 11},
      {"cudaErrorInvalidDevicePointer", 17}, {"cudaErrorInvalidMemcpyDirection", 21},
      {"cudaErrorInvalidResourceHandle", 33}, {"cudaErrorNotReady", 34},
      {"cudaDevAttrMaxThreadsPerBlock", 1}, {"cudaDevAttrWarpSize", 10},
      {"cudaDevAttrComputeCapabilityMajor", 75}, {"cudaDevAttrComputeCapabilityMinor", 76},
      {"NULL", 0}};
  return m;
}

const char* spaceName(int s) {
  switch (s) {
    case 0: return "__host__";
    case 1: return "__device__";
    case 2: return "__host__ __device__";
    default: return "__global__";
  }
}

bool deviceCtx(int s) { return s != 0; }

class Lowerer {
 public:
  Lowerer(std::shared_ptr<Unit> u, Program& p) : u_(std::move(u)), P_(p) {}

  void run() {
    P_.sharedDefaultName = P_.intern("(dynamic shared)");
    checkFunctions();
    for (auto& g : u_->globals) lowerGlobal(g);
    // function metadata first (calls may refer forward)
    P_.fns.resize(u_->fns.size());
    for (size_t i = 0; i < u_->fns.size(); ++i) P_.fnNames.push_back(u_->fns[i].name);
    for (size_t i = 0; i < u_->fns.size(); ++i) lowerFunction(static_cast<int>(i));
    P_.mainIndex = mainIndex_;
  }

 private:
  std::shared_ptr<Unit> u_;
  Program& P_;
  int mainIndex_ = -1;

  struct Var { int slot; Ty ty; };
  std::vector<std::map<std::string, Var>> scopes_;
  Function* fn_ = nullptr;
  int fnIndex_ = -1;
  int nSlots_ = 0;
  std::vector<mck_local> fnLocals_;

  // loop context for break/continue
  struct Loop {
    int scopeDepth;              // scopes open when the loop frame was pushed
    std::vector<int> breaks;     // pcs to patch with the exit
    std::vector<int> continues;  // pcs to patch with the continue target
  };
  std::vector<Loop> loops_;
  int scopeDepth_ = 0;  // run-time scopes open inside the current function body

  // ---------------- checks ----------------
  void checkFunctions() {
    int count = 0;
    Pos last{1, 1};
    for (size_t i = 0; i < u_->fns.size(); ++i) {
      Function& f = u_->fns[i];
      if (f.name != "main" || !f.body) continue;
      ++count;
      last = f.pos;
      mainIndex_ = static_cast<int>(i);
      if (!(f.ret.base == MCK_INT && f.ret.ptr == 0 && !f.ret.isArray())) semErr(f.pos, "'main' must return int");
      if (!f.params.empty()) semErr(f.pos, "'main' must take no parameters");
      if (f.space != 0) semErr(f.pos, "'main' cannot carry execution-space attributes");
    }
    if (count == 0) semErr(u_->fns.empty() ? Pos{1, 1} : u_->fns[0].pos, "program has no 'main' function");
    if (count > 1) semErr(last, "program has more than one 'main' function");
    for (size_t i = 0; i < u_->fns.size(); ++i)
      for (size_t j = i + 1; j < u_->fns.size(); ++j)
        if (u_->fns[i].name == u_->fns[j].name && u_->fns[i].body && u_->fns[j].body)
          semErr(u_->fns[j].pos, "redefinition of function '" + u_->fns[j].name + "'");
    for (auto& f : u_->fns)
      if (f.space == 3 && !f.ret.isVoid()) semErr(f.pos, "__global__ function '" + f.name + "' must return void");
  }

  void lowerGlobal(GlobalDef& g) {
    if (g.ty.isVoid()) semErr(g.pos, "variable '" + g.name + "' declared void");
    if (g.init) {
      const Expr* e = g.init;
      if (e->k == EK::Int) {
        g.ival = e->ival;
        g.hasInit = true;
      } else if (e->k == EK::Flt) {
        g.fval = e->fval;
        g.ival = static_cast<int64_t>(e->fval);
        g.hasInit = true;
      } else if (e->k == EK::Un && e->op == MCK_NEG && e->a->k == EK::Int) {
        g.ival = -e->a->ival;
        g.hasInit = true;
      } else {
        semErr(e->pos, "global initializer must be a constant");
      }
    }
    GlobalInfo gi;
    gi.name = g.name;
    gi.type = g.ty.code();
    gi.size = g.ty.bytes();
    gi.device = g.device;
    gi.hasInit = g.hasInit;
    gi.ival = g.ival;
    gi.fval = g.fval;
    P_.globals.push_back(gi);
  }

  int findFunction(const std::string& n) const {
    int proto = -1;
    for (size_t i = 0; i < u_->fns.size(); ++i) {
      if (u_->fns[i].name != n) continue;
      if (u_->fns[i].body) return static_cast<int>(i);
      proto = static_cast<int>(i);
    }
    return proto;
  }
  int findGlobal(const std::string& n) const {
    for (size_t i = 0; i < u_->globals.size(); ++i)
      if (u_->globals[i].name == n) return static_cast<int>(i);
    return -1;
  }
  std::optional<Var> lookup(const std::string& n) const {
    for (auto it = scopes_.rbegin(); it != scopes_.rend(); ++it) {
      auto f = it->find(n);
      if (f != it->end()) return f->second;
    }
    return std::nullopt;
  }
  int declare(const std::string& name, const Ty& ty, Pos pos, bool param, bool dyn) {
    if (ty.isVoid()) semErr(pos, param ? "parameter declared void" : "variable '" + name + "' declared void");
    if (scopes_.back().count(name))
      semErr(pos, param ? "duplicate parameter '" + name + "'" : "redeclaration of '" + name + "' in the same scope");
    int slot = nSlots_++;
    scopes_.back()[name] = Var{slot, ty};
    mck_local l{};
    l.size = static_cast<int32_t>(ty.bytes());
    l.name = P_.intern(name);
    l.type = ty.code();
    l.is_param = param ? 1 : 0;
    l.is_dyn_shared = dyn ? 1 : 0;
    fnLocals_.push_back(l);
    return slot;
  }

  // ---------------- emission ----------------
  int pc() const { return static_cast<int>(P_.code.size()); }
  int emit(int op, int line, int a = 0, int b = 0, uint8_t t = 0, uint8_t f = 0) {
    mck_ins in{};
    in.op = static_cast<uint8_t>(op);
    in.t = t;
    in.f = f;
    in.a = a;
    in.b = b;
    in.line = line;
    P_.code.push_back(in);
    return pc() - 1;
  }
  void patch(int at, int target) { P_.code[static_cast<size_t>(at)].a = target; }

  void lowerFunction(int idx) {
    Function& f = u_->fns[static_cast<size_t>(idx)];
    mck_fn& m = P_.fns[static_cast<size_t>(idx)];
    m.entry = -1;
    m.ret = f.ret.code();
    m.space = static_cast<uint8_t>(f.space);
    m.n_params = static_cast<int32_t>(f.params.size());
    m.dyn_shared_slot = -1;
    m.local_base = static_cast<int32_t>(P_.locals.size());
    if (!f.body) return;
    fn_ = &f;
    fnIndex_ = idx;
    nSlots_ = 0;
    fnLocals_.clear();
    scopes_.clear();
    scopes_.emplace_back();
    loops_.clear();
    scopeDepth_ = 0;
    for (auto& p : f.params) declare(p.name, p.ty, p.pos, true, false);
    m.entry = pc();
    stmt(f.body);
    emit(OP_FALLOFF, f.body->pos.line, 0, 0, f.ret.code());
    scopes_.pop_back();
    m.n_slots = nSlots_;
    for (size_t i = 0; i < fnLocals_.size(); ++i)
      if (fnLocals_[i].is_dyn_shared) m.dyn_shared_slot = static_cast<int32_t>(i);
    P_.locals.insert(P_.locals.end(), fnLocals_.begin(), fnLocals_.end());
    fn_ = nullptr;
  }

  static bool lvalueForm(const Expr* e) {
    if (e->k == EK::Name) return e->bind == Bind::Local || e->bind == Bind::Global;
    return e->k == EK::Idx || (e->k == EK::Un && e->op == 10);
  }
  static bool lvalueSyntax(const Expr* e) {
    return e->k == EK::Name || e->k == EK::Idx || (e->k == EK::Un && e->op == 10);
  }

  void stmt(Stmt* s) {
    const int L = s->pos.line;
    switch (s->k) {
      case SK::Block: {
        scopes_.emplace_back();
        emit(OP_SCOPE_PUSH, L);
        ++scopeDepth_;
        for (Stmt* c : s->body) stmt(c);
        --scopeDepth_;
        emit(OP_SCOPE_POP, L);
        scopes_.pop_back();
        break;
      }
      case SK::If: {
        resolve(s->cond);
        emit(OP_NOP, L);
        rv(s->cond);
        int judge = emit(OP_IFJUDGE, L);
        stmt(s->thenS);
        if (s->elseS) {
          int j = emit(OP_JMP, L);
          patch(judge, pc());
          stmt(s->elseS);
          patch(j, pc());
        } else {
          patch(judge, pc());
        }
        break;
      }
      case SK::While: {
        resolve(s->cond);
        emit(OP_NOP, L);
        int condPc = pc();
        rv(s->cond);
        int judge = emit(OP_WHILEJUDGE, L);
        loops_.push_back(Loop{scopeDepth_, {}, {}});
        stmt(s->loop);
        emit(OP_JMP, L, condPc);
        int exit = pc();
        patch(judge, exit);
        for (int b : loops_.back().breaks) patch(b, exit);
        for (int c : loops_.back().continues) patch(c, condPc);
        loops_.pop_back();
        break;
      }
      case SK::For: {
        scopes_.emplace_back();
        emit(OP_SCOPE_PUSH, L);
        ++scopeDepth_;
        if (s->init && s->init->k != SK::Empty) stmt(s->init);
        if (s->cond) resolve(s->cond);
        if (s->incr) resolve(s->incr);
        int condPc = pc();
        if (s->cond) rv(s->cond);
        int judge = emit(OP_FORJUDGE, L, 0, 0, 0, s->cond ? 1 : 0);
        loops_.push_back(Loop{scopeDepth_, {}, {}});
        stmt(s->loop);
        int contPc = pc();
        if (s->incr) {
          rv(s->incr);
          emit(OP_POPVALUE, L);
        }
        emit(OP_JMP, L, condPc);
        --scopeDepth_;
        int exit = emit(OP_SCOPE_POP, L);
        patch(judge, exit);
        for (int b : loops_.back().breaks) patch(b, exit);
        for (int c : loops_.back().continues) patch(c, contPc);
        loops_.pop_back();
        scopes_.pop_back();
        break;
      }
      case SK::Ret:
        if (s->e) {
          if (fn_->ret.isVoid()) semErr(s->pos, "void function '" + fn_->name + "' returns a value");
          resolve(s->e);
          emit(OP_NOP, L);
          rv(s->e);
          emit(OP_RETURN, L, 0, 0, fn_->ret.code(), 1);
        } else {
          if (!fn_->ret.isVoid() && fn_->name != "main")
            semErr(s->pos, "non-void function '" + fn_->name + "' returns no value");
          emit(OP_NOP, L);
          emit(OP_RETURN, L, 0, 0, fn_->ret.code(), 0);
        }
        break;
      case SK::Brk: {
        if (loops_.empty()) semErr(s->pos, "'break' outside of a loop");
        int at = emit(OP_BREAK, L, 0, scopeDepth_ - loops_.back().scopeDepth);
        loops_.back().breaks.push_back(at);
        break;
      }
      case SK::Cont: {
        if (loops_.empty()) semErr(s->pos, "'continue' outside of a loop");
        int at = emit(OP_CONTINUE, L, 0, scopeDepth_ - loops_.back().scopeDepth);
        loops_.back().continues.push_back(at);
        break;
      }
      case SK::ExprS:
        resolve(s->e);
        emit(OP_NOP, L);
        rv(s->e);
        emit(OP_POPVALUE, L);
        break;
      case SK::Decl: {
        if (s->externShared) {
          if (fn_->space != 3) semErr(s->pos, "extern __shared__ is only valid inside a __global__ kernel");
          emit(OP_NOP, L);
          for (auto& d : s->decls) {
            if (!fn_->dynSharedName.empty())
              semErr(d.pos, "kernel '" + fn_->name + "' already has a dynamic shared array '" +
                                fn_->dynSharedName + "'");
            d.slot = declare(d.name, d.ty, d.pos, false, true);
            fn_->dynSharedName = d.name;
            if (d.init) semErr(d.pos, "extern __shared__ arrays cannot have initializers");
            emit(OP_DECL, d.pos.line, d.slot, 0, d.ty.code(), 1);
          }
          emit(OP_NOP, L);
          break;
        }
        emit(OP_NOP, L);
        for (auto& d : s->decls) {
          d.slot = declare(d.name, d.ty, d.pos, false, false);
          if (d.init) resolve(d.init);
          if (d.init && d.ty.isArray()) semErr(d.pos, "array '" + d.name + "' cannot have a scalar initializer");
          emit(OP_DECL, d.pos.line, d.slot, 0, d.ty.code(), 0);
          if (d.init) {
            rv(d.init);
            emit(OP_INITSTORE, d.pos.line, d.slot, 0, d.ty.code());
          }
        }
        emit(OP_NOP, L);
        break;
      }
      case SK::Empty:
        emit(OP_NOP, L);
        break;
    }
  }

  // ---------------- expressions: resolution (lower.cpp rules) ----------------
  void resolve(Expr* e) {
    switch (e->k) {
      case EK::Int: case EK::Flt: case EK::Builtin: break;
      case EK::Str: semErr(e->pos, "string literals may only appear as the first argument of printf");
      case EK::Name: resolveName(e); break;
      case EK::Mem: resolveMember(e); break;
      case EK::Un:
        resolve(e->a);
        if (e->op == 11 && !lvalueSyntax(e->a)) semErr(e->pos, "cannot take the address of this expression");
        if (e->op == 11 && e->a->k == EK::Name && e->a->bind == Bind::Func)
          semErr(e->pos, "function pointers are not supported");
        break;
      case EK::IncDec:
        resolve(e->a);
        assignable(e->a, e->pos);
        break;
      case EK::Bin: resolve(e->a); resolve(e->b); break;
      case EK::Asg:
        resolve(e->a);
        resolve(e->b);
        assignable(e->a, e->pos);
        break;
      case EK::Cond: resolve(e->a); resolve(e->b); resolve(e->c); break;
      case EK::Cast: resolve(e->a); break;
      case EK::Sizeof:
        if (e->a) {
          resolve(e->a);
          e->castTy = typeOf(e->a, e->pos);
        }
        break;
      case EK::Idx: resolve(e->a); resolve(e->b); break;
      case EK::Call: resolveCall(e); break;
      case EK::Launch: resolveLaunch(e); break;
    }
  }

  void assignable(const Expr* t, Pos p) {
    if (!lvalueSyntax(t)) semErr(p, "assignment target is not an lvalue");
    if (t->k == EK::Name) {
      if (t->bind == Bind::Func || t->bind == Bind::Enum) semErr(p, "'" + t->text + "' is not assignable");
      Ty ty = t->bind == Bind::Local ? t->lit : t->bind == Bind::Global ? u_->globals[t->index].ty : Ty{};
      if (ty.isArray()) semErr(p, "array '" + t->text + "' is not assignable");
    }
  }

  void resolveName(Expr* e) {
    if (auto v = lookup(e->text)) {
      e->bind = Bind::Local;
      e->index = v->slot;
      e->lit = v->ty;
      return;
    }
    int g = findGlobal(e->text);
    if (g >= 0) {
      e->bind = Bind::Global;
      e->index = g;
      return;
    }
    if (e->text == "warpSize") {
      if (!deviceCtx(fn_->space)) semErr(e->pos, "'warpSize' is only available in device code");
      e->k = EK::Builtin;
      e->builtin = MCK_B_WARP;
      e->comp = 0;
      return;
    }
    auto c = enumConsts().find(e->text);
    if (c != enumConsts().end()) {
      e->bind = Bind::Enum;
      e->cval = c->second;
      return;
    }
    int f = findFunction(e->text);
    if (f >= 0) {
      e->bind = Bind::Func;
      e->index = f;
      return;
    }
    semErr(e->pos, "use of undeclared identifier '" + e->text + "'");
  }

  void resolveMember(Expr* e) {
    static const std::map<std::string, int> vars = {
        {"threadIdx", MCK_B_TID}, {"blockIdx", MCK_B_BID}, {"blockDim", MCK_B_BDIM}, {"gridDim", MCK_B_GDIM}};
    if (e->a->k != EK::Name) semErr(e->pos, "member access is only supported on CUDA builtins");
    auto it = vars.find(e->a->text);
    if (it == vars.end())
      semErr(e->pos, "member access is only supported on CUDA builtins (structs are not supported)");
    if (!deviceCtx(fn_->space)) semErr(e->pos, "'" + e->a->text + "' is only available in device code");
    int comp;
    if (e->text == "x") comp = 0;
    else if (e->text == "y") comp = 1;
    else if (e->text == "z") comp = 2;
    else semErr(e->pos, "unknown component '." + e->text + "' on '" + e->a->text + "'");
    e->text = e->a->text + "." + e->text;
    e->k = EK::Builtin;
    e->builtin = it->second;
    e->comp = comp;
    e->a = nullptr;
  }

  static bool calleeOk(int caller, int callee) {
    switch (caller) {
      case 0: return callee == 0 || callee == 2;
      case 1: case 3: return callee == 1 || callee == 2;
      default: return callee == 2;
    }
  }

  void resolveCall(Expr* e) {
    if (e->a->k != EK::Name) semErr(e->pos, "only direct calls of named functions are supported");
    const std::string& n = e->a->text;
    if (lookup(n)) semErr(e->pos, "'" + n + "' is not a function");
    if (n == "printf") {
      if (fn_->space != 0) semErr(e->pos, "printf is only supported in host code");
      if (e->args.empty() || e->args[0]->k != EK::Str)
        semErr(e->pos, "printf requires a string literal format as its first argument");
      e->callee = Callee::Printf;
      e->args[0]->strId = static_cast<int>(P_.strings.size());
      P_.strings.push_back(e->args[0]->sval);  // not interned: one entry per format
      for (size_t i = 1; i < e->args.size(); ++i) resolve(e->args[i]);
      return;
    }
    static const std::map<std::string, std::pair<int, int>> syncs = {
        {"__syncthreads", {MCK_SYNC_PLAIN, 0}}, {"__syncthreads_and", {MCK_SYNC_AND, 1}},
        {"__syncthreads_or", {MCK_SYNC_OR, 1}}, {"__syncthreads_count", {MCK_SYNC_COUNT, 1}}};
    auto sy = syncs.find(n);
    if (sy != syncs.end()) {
      if (fn_->space != 3 && fn_->space != 1) semErr(e->pos, "'" + n + "' may only be called from device code");
      if (static_cast<int>(e->args.size()) != sy->second.second)
        semErr(e->pos, "'" + n + "' takes " + std::to_string(sy->second.second) + " argument(s)");
      e->callee = Callee::Sync;
      e->syncKind = sy->second.first;
      for (Expr* a : e->args) resolve(a);
      return;
    }
    auto api = apis().find(n);
    if (api != apis().end()) {
      if (fn_->space != 0) semErr(e->pos, "CUDA runtime API call '" + n + "' is only allowed in host code");
      int k = static_cast<int>(e->args.size());
      if (k < api->second.mn || k > api->second.mx) semErr(e->pos, "wrong number of arguments to '" + n + "'");
      e->callee = Callee::Api;
      e->calleeIndex = api->second.id;
      for (Expr* a : e->args) resolve(a);
      return;
    }
    if (n.compare(0, 4, "cuda") == 0) semErr(e->pos, "unsupported CUDA runtime API function '" + n + "'");
    int f = findFunction(n);
    if (f < 0) semErr(e->pos, "call to undeclared function '" + n + "'");
    const Function& c = u_->fns[static_cast<size_t>(f)];
    if (!calleeOk(fn_->space, c.space)) {
      if (c.space == 3) semErr(e->pos, "kernel '" + n + "' must be launched with <<<...>>>");
      semErr(e->pos, std::string("function '") + n + "' (" + spaceName(c.space) + ") cannot be called from " +
                         spaceName(fn_->space) + " function '" + fn_->name + "'");
    }
    if (e->args.size() != c.params.size())
      semErr(e->pos, "wrong number of arguments to '" + n + "' (expected " + std::to_string(c.params.size()) + ")");
    if (!c.body) semErr(e->pos, "call of '" + n + "', which has no definition");
    e->callee = Callee::User;
    e->calleeIndex = f;
    e->a->bind = Bind::Func;
    e->a->index = f;
    for (Expr* a : e->args) resolve(a);
  }

  void resolveLaunch(Expr* e) {
    if (fn_->space != 0) semErr(e->pos, "kernel launches are only allowed in host code");
    if (e->a->k != EK::Name) semErr(e->pos, "launch target must be a kernel name");
    int f = findFunction(e->a->text);
    if (f < 0) semErr(e->pos, "launch of undeclared function '" + e->a->text + "'");
    const Function& k = u_->fns[static_cast<size_t>(f)];
    if (k.space != 3) semErr(e->pos, "'" + e->a->text + "' is not a __global__ kernel");
    if (!k.body) semErr(e->pos, "launch of kernel '" + e->a->text + "' with no definition");
    if (e->args.size() != k.params.size())
      semErr(e->pos, "wrong number of arguments to kernel '" + e->a->text + "' (expected " +
                         std::to_string(k.params.size()) + ")");
    e->callee = Callee::User;
    e->calleeIndex = f;
    e->a->bind = Bind::Func;
    e->a->index = f;
    resolve(e->grid);
    resolve(e->block);
    if (e->shmem) resolve(e->shmem);
    if (e->stream) resolve(e->stream);
    for (Expr* a : e->args) resolve(a);
  }

  Ty typeOf(const Expr* e, Pos p) {
    Ty intT;
    switch (e->k) {
      case EK::Int: case EK::Flt: return e->lit;
      case EK::Str: { Ty t; t.base = MCK_CHAR; t.ptr = 1; return t; }
      case EK::Name:
        if (e->bind == Bind::Local) return e->lit;
        if (e->bind == Bind::Global) return u_->globals[static_cast<size_t>(e->index)].ty;
        if (e->bind == Bind::Enum) return intT;
        semErr(p, "cannot take the size of this expression");
      case EK::Builtin: return intT;
      case EK::Un:
        if (e->op == 10) {
          Ty t = typeOf(e->a, p);
          if (t.isArray()) { t.arr = -1; ++t.ptr; }
          if (t.isArray()) t.arr = -1; else --t.ptr;
          return t;
        }
        if (e->op == 11) {
          Ty t = typeOf(e->a, p);
          ++t.ptr;
          return t;
        }
        return typeOf(e->a, p);
      case EK::IncDec: return typeOf(e->a, p);
      case EK::Bin: {
        Ty l = typeOf(e->a, p), r = typeOf(e->b, p);
        if (l.isArray()) { l.arr = -1; ++l.ptr; }
        if (r.isArray()) { r.arr = -1; ++r.ptr; }
        if (e->op >= MCK_LT && e->op <= MCK_NE) return intT;
        if (e->op == MCK_LAND || e->op == MCK_LOR) return intT;
        if (l.ptr > 0) return l;
        if (r.ptr > 0) return r;
        Ty t;
        if (l.base == MCK_DOUBLE || r.base == MCK_DOUBLE) t.base = MCK_DOUBLE;
        else if (l.base == MCK_FLOAT || r.base == MCK_FLOAT) t.base = MCK_FLOAT;
        else if (l.base == MCK_LONG || r.base == MCK_LONG) t.base = MCK_LONG;
        else if (l.base == MCK_UINT || r.base == MCK_UINT) t.base = MCK_UINT;
        return t;
      }
      case EK::Asg: return typeOf(e->a, p);
      case EK::Cond: return typeOf(e->b, p);
      case EK::Cast: return e->castTy;
      case EK::Sizeof: { Ty t; t.base = MCK_LONG; return t; }
      case EK::Idx: {
        Ty t = typeOf(e->a, p);
        if (t.isArray()) { t.arr = -1; ++t.ptr; }
        --t.ptr;
        return t;
      }
      case EK::Call:
        if (e->callee == Callee::User) return u_->fns[static_cast<size_t>(e->calleeIndex)].ret;
        return intT;
      default: { Ty t; t.base = MCK_VOID; return t; }
    }
  }

  // ---------------- expressions: code ----------------
  void rv(Expr* e) {
    ex(e);
    if (lvalueForm(e)) emit(OP_LOADRV, e->pos.line);
  }

  void ex(Expr* e) {
    const int L = e->pos.line;
    switch (e->k) {
      case EK::Int: {
        uint64_t v = static_cast<uint64_t>(e->ival);
        emit(OP_PUSH_INT, L, static_cast<int32_t>(v & 0xffffffffu), static_cast<int32_t>(v >> 32), e->lit.code());
        break;
      }
      case EK::Flt: {
        union { double d; uint64_t u; } c;
        c.d = e->fval;
        emit(OP_PUSH_FLT, L, static_cast<int32_t>(c.u & 0xffffffffu), static_cast<int32_t>(c.u >> 32), e->lit.code());
        break;
      }
      case EK::Str: emit(OP_UB, L, MCK_UB_STRLIT); break;
      case EK::Name:
        if (e->bind == Bind::Local) {
          emit(OP_PUSH_LOCAL, L, e->index, P_.intern(e->text), e->lit.code());
        } else if (e->bind == Bind::Global) {
          emit(OP_PUSH_GLOBAL, L, e->index, 0, u_->globals[static_cast<size_t>(e->index)].ty.code());
        } else if (e->bind == Bind::Enum) {
          uint64_t v = static_cast<uint64_t>(e->cval);
          emit(OP_PUSH_INT, L, static_cast<int32_t>(v & 0xffffffffu), static_cast<int32_t>(v >> 32), MCK_T_INT);
        } else {
          emit(OP_UB, L, MCK_UB_NOVALUE, P_.intern(e->text));
        }
        break;
      case EK::Builtin: emit(OP_PUSH_BUILTIN, L, e->comp, P_.intern(e->text), 0, static_cast<uint8_t>(e->builtin)); break;
      case EK::Mem: emit(OP_UB, L, MCK_UB_MEMBER); break;
      case EK::Un:
        emit(OP_NOP, L);
        if (e->op == 10) {
          rv(e->a);
          emit(OP_DEREF, L);
        } else if (e->op == 11) {
          ex(e->a);
          emit(OP_ADDROF, L);
        } else {
          rv(e->a);
          emit(OP_UNARY, L, 0, 0, 0, static_cast<uint8_t>(e->op));
        }
        break;
      case EK::IncDec:
        emit(OP_NOP, L);
        ex(e->a);
        emit(OP_LOADKEEP, L);
        emit(OP_STORE_INC, L, e->delta, 0, 0, e->prefix ? 1 : 0);
        break;
      case EK::Bin:
        emit(OP_NOP, L);
        if (e->op == MCK_LAND || e->op == MCK_LOR) {
          rv(e->a);
          int j = emit(OP_LOGRHS, L, 0, 0, 0, e->op == MCK_LAND ? 1 : 0);
          rv(e->b);
          emit(OP_BOOLIFY, L);
          patch(j, pc());
        } else {
          rv(e->a);
          rv(e->b);
          emit(OP_BINARY, L, 0, 0, 0, static_cast<uint8_t>(e->op));
        }
        break;
      case EK::Asg:
        emit(OP_NOP, L);
        ex(e->a);
        if (e->compound) {
          emit(OP_LOADKEEP, L);
          rv(e->b);
          emit(OP_STORE_OP, L, 0, 0, 0, static_cast<uint8_t>(e->op));
        } else {
          rv(e->b);
          emit(OP_STORE, L);
        }
        break;
      case EK::Cond: {
        emit(OP_NOP, L);
        rv(e->a);
        int sel = emit(OP_TERNSEL, L);
        rv(e->b);
        int j = emit(OP_JMP, L);
        patch(sel, pc());
        rv(e->c);
        patch(j, pc());
        break;
      }
      case EK::Call: {
        emit(OP_NOP, L);
        size_t first = e->callee == Callee::Printf ? 1 : 0;
        for (size_t i = first; i < e->args.size(); ++i) rv(e->args[i]);
        int n = static_cast<int>(e->args.size() - first);
        switch (e->callee) {
          case Callee::User: emit(OP_CALL, L, e->calleeIndex, n); break;
          case Callee::Printf: emit(OP_PRINTF, L, e->args[0]->strId, n); break;
          case Callee::Api: emit(OP_API, L, e->calleeIndex, n); break;
          case Callee::Sync: emit(OP_SYNC, L, 0, 0, 0, static_cast<uint8_t>(e->syncKind)); break;
          case Callee::None: emit(OP_UB, L, MCK_UB_NOCALL); break;
        }
        break;
      }
      case EK::Idx:
        emit(OP_NOP, L);
        rv(e->a);
        rv(e->b);
        emit(OP_INDEX, L);
        break;
      case EK::Cast:
        emit(OP_NOP, L);
        rv(e->a);
        emit(OP_CAST, L, 0, 0, e->castTy.code());
        break;
      case EK::Sizeof: {
        uint64_t v = static_cast<uint64_t>(e->castTy.bytes());
        emit(OP_PUSH_INT, L, static_cast<int32_t>(v & 0xffffffffu), static_cast<int32_t>(v >> 32), MCK_T_LONG);
        break;
      }
      case EK::Launch: {
        emit(OP_NOP, L);
        rv(e->grid);
        rv(e->block);
        if (e->shmem) rv(e->shmem);
        if (e->stream) rv(e->stream);
        for (Expr* a : e->args) rv(a);
        emit(OP_LAUNCH, L, e->calleeIndex, static_cast<int>(e->args.size()), 0,
             static_cast<uint8_t>((e->shmem ? 1 : 0) | (e->stream ? 2 : 0)));
        break;
      }
    }
  }
};

const char* opName(int op) {
  static const char* n[] = {"nop", "scope_push", "scope_pop", "jmp", "push_int", "push_flt",
                            "push_local", "push_global", "push_builtin", "ub", "loadrv",
                            "loadkeep", "store", "store_op", "store_inc", "addrof", "deref",
                            "index", "unary", "binary", "logrhs", "boolify", "ternsel", "cast",
                            "ifjudge", "whilejudge", "forjudge", "popvalue", "return", "break",
                            "continue", "call", "falloff", "sync", "decl", "initstore", "printf",
                            "api", "launch"};
  return op < OP_COUNT ? n[op] : "?";
}

}  // namespace

std::string Program::disassemble() const {
  std::string out;
  char buf[160];
  for (size_t f = 0; f < fns.size(); ++f) {
    std::snprintf(buf, sizeof buf, "fn %zu %s entry=%d slots=%d params=%d space=%d\n", f,
                  fnNames[f].c_str(), fns[f].entry, fns[f].n_slots, fns[f].n_params, fns[f].space);
    out += buf;
  }
  for (size_t i = 0; i < code.size(); ++i) {
    const mck_ins& c = code[i];
    std::snprintf(buf, sizeof buf, "%5zu  %-12s t=%02x f=%d a=%d b=%d  line %d\n", i, opName(c.op), c.t,
                  c.f, c.a, c.b, c.line);
    out += buf;
  }
  return out;
}

std::shared_ptr<const Program> compileProgram(const std::string& source, const std::string& filename) {
  auto p = std::make_shared<Program>();
  p->unit = parseUnit(source, filename);
  p->filename = filename;
  Lowerer l(p->unit, *p);
  l.run();
  return p;
}

}  // namespace mckb
