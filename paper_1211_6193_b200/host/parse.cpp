// parse.cpp -- tokenizer, object-like-macro preprocessor and recursive-descent
// parser for the CUDA-C subset.
//
// Provenance: this front end restates /root/reference/proj/src/lexer.cpp and
// parser.cpp closely -- the same grammar, the same precedence and
// compound-assignment tables, the same production order -- because its
// outputs (accepted language, node positions, error texts) must be
// byte-identical to the reference's.  It runs once per program on the host,
// outside the B200 hot path, and is not claimed as new work.
#include <cctype>
#include <cerrno>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "ast.hpp"
#include "mck_ir.h"

namespace mckb {

int64_t Ty::scalar() const {
  if (ptr > 0) return 8;
  switch (base) {
    case MCK_CHAR: return 1;
    case MCK_INT: case MCK_UINT: case MCK_FLOAT: return 4;
    case MCK_LONG: case MCK_DOUBLE: return 8;
    default: return 0;
  }
}

uint8_t Ty::code() const { return MCK_T(base, ptr, isArray() ? 1 : 0); }

namespace {

enum T {
  tEnd, tId, tInt, tFlt, tChr, tStr,
  // keywords
  kVoid, kChar, kInt, kUnsigned, kLong, kFloat, kDouble, kIf, kElse, kWhile, kFor, kReturn,
  kBreak, kContinue, kSizeof, kExtern, kGlobal, kDevice, kHost, kShared, kNoinline, kForceinline,
  // punctuation
  pLP, pRP, pLB, pRB, pLS, pRS, pSemi, pComma, pDot, pArrow, pQ, pColon, pPlus, pMinus, pStar,
  pSlash, pPct, pInc, pDec, pAmp, pPipe, pCaret, pTilde, pBang, pAndAnd, pOrOr, pShl, pShr, pLt,
  pLe, pGt, pGe, pEq, pNe, pAsg, pAddA, pSubA, pMulA, pDivA, pRemA, pShlA, pShrA, pAndA, pOrA,
  pXorA, pLaunchOpen, pLaunchClose
};

struct Tok {
  T k = tEnd;
  Pos pos;
  std::string text;
  std::string sval;
  int64_t ival = 0;
  double fval = 0;
  bool isU = false, isL = false, isF = false;
};

const char* tokDesc(T k) {
  static const char* names[] = {
      "end of input", "identifier", "integer literal", "float literal", "character literal",
      "string literal", "'void'", "'char'", "'int'", "'unsigned'", "'long'", "'float'",
      "'double'", "'if'", "'else'", "'while'", "'for'", "'return'", "'break'", "'continue'",
      "'sizeof'", "'extern'", "'__global__'", "'__device__'", "'__host__'", "'__shared__'",
      "'__noinline__'", "'__forceinline__'", "'('", "')'", "'{'", "'}'", "'['", "']'", "';'",
      "','", "'.'", "'->'", "'?'", "':'", "'+'", "'-'", "'*'", "'/'", "'%'", "'++'", "'--'",
      "'&'", "'|'", "'^'", "'~'", "'!'", "'&&'", "'||'", "'<<'", "'>>'", "'<'", "'<='", "'>'",
      "'>='", "'=='", "'!='", "'='", "'+='", "'-='", "'*='", "'/='", "'%='", "'<<='", "'>>='",
      "'&='", "'|='", "'^='", "'<<<'", "'>>>'"};
  return names[k];
}

[[noreturn]] void fail(const char* stage, Pos p, const std::string& m) {
  throw FrontendFailure{stage, p, m};
}

const std::map<std::string, T>& keywords() {
  static const std::map<std::string, T> m = {
      {"void", kVoid}, {"char", kChar}, {"int", kInt}, {"unsigned", kUnsigned},
      {"long", kLong}, {"float", kFloat}, {"double", kDouble}, {"if", kIf}, {"else", kElse},
      {"while", kWhile}, {"for", kFor}, {"return", kReturn}, {"break", kBreak},
      {"continue", kContinue}, {"sizeof", kSizeof}, {"extern", kExtern}, {"__global__", kGlobal},
      {"__device__", kDevice}, {"__host__", kHost}, {"__shared__", kShared},
      {"__noinline__", kNoinline}, {"__forceinline__", kForceinline}};
  return m;
}

// Character scanner over one buffer.
struct Scan {
  const std::string& s;
  size_t i = 0;
  int line = 1, col = 1;
  explicit Scan(const std::string& src) : s(src) {}
  bool end() const { return i >= s.size(); }
  char c(size_t k = 0) const { return i + k < s.size() ? s[i + k] : '\0'; }
  void adv() {
    ++i;
    ++col;
  }
  Pos here() const { return Pos{line, col}; }
  void skip() {
    while (!end()) {
      char ch = c();
      if (ch == '\n') {
        ++i;
        ++line;
        col = 1;
      } else if (isspace((unsigned char)ch)) {
        adv();
      } else if (ch == '/' && c(1) == '/') {
        while (!end() && c() != '\n') adv();
      } else if (ch == '/' && c(1) == '*') {
        Pos st = here();
        adv();
        adv();
        while (!end() && !(c() == '*' && c(1) == '/')) {
          if (c() == '\n') {
            ++i;
            ++line;
            col = 1;
          } else {
            adv();
          }
        }
        if (end()) fail("lex", st, "unterminated comment");
        adv();
        adv();
      } else {
        break;
      }
    }
  }
  Tok ident() {
    Tok t;
    t.pos = here();
    size_t b = i;
    while (!end() && (isalnum((unsigned char)c()) || c() == '_')) adv();
    t.text = s.substr(b, i - b);
    auto it = keywords().find(t.text);
    t.k = it == keywords().end() ? tId : it->second;
    return t;
  }
  void intSuffix(Tok& t) {
    while (c() == 'u' || c() == 'U' || c() == 'l' || c() == 'L') {
      if (c() == 'u' || c() == 'U') t.isU = true;
      else t.isL = true;
      adv();
    }
  }
  Tok number() {
    Tok t;
    t.pos = here();
    size_t b = i;
    if (c() == '0' && (c(1) == 'x' || c(1) == 'X')) {
      adv();
      adv();
      while (isxdigit((unsigned char)c())) adv();
      t.k = tInt;
      t.text = s.substr(b, i - b);
      t.ival = (int64_t)strtoull(t.text.c_str(), nullptr, 16);
      intSuffix(t);
      return t;
    }
    bool flt = false;
    while (isdigit((unsigned char)c())) adv();
    if (c() == '.' && isdigit((unsigned char)c(1))) {
      flt = true;
      adv();
      while (isdigit((unsigned char)c())) adv();
    }
    if (c() == 'e' || c() == 'E') {
      size_t save = i;
      int scol = col;
      adv();
      if (c() == '+' || c() == '-') adv();
      if (isdigit((unsigned char)c())) {
        flt = true;
        while (isdigit((unsigned char)c())) adv();
      } else {
        i = save;
        col = scol;
      }
    }
    t.text = s.substr(b, i - b);
    if (flt) {
      t.k = tFlt;
      t.fval = strtod(t.text.c_str(), nullptr);
      if (c() == 'f' || c() == 'F') {
        t.isF = true;
        adv();
      }
    } else {
      t.k = tInt;
      errno = 0;
      t.ival = strtoll(t.text.c_str(), nullptr, 10);
      if (errno == ERANGE) fail("lex", t.pos, "integer literal out of range");
      intSuffix(t);
    }
    return t;
  }
  char escape(Pos st) {
    adv();
    char ch = c();
    adv();
    switch (ch) {
      case 'n': return '\n';
      case 't': return '\t';
      case 'r': return '\r';
      case '0': return '\0';
      case '\\': return '\\';
      case '\'': return '\'';
      case '"': return '"';
      default: fail("lex", st, std::string("unknown escape sequence '\\") + ch + "'");
    }
  }
  Tok chr() {
    Tok t;
    t.pos = here();
    t.k = tChr;
    adv();
    if (end() || c() == '\n') fail("lex", t.pos, "unterminated character literal");
    char v;
    if (c() == '\\') {
      v = escape(t.pos);
    } else {
      v = c();
      adv();
    }
    if (c() != '\'') fail("lex", t.pos, "unterminated character literal");
    adv();
    t.ival = (int64_t)v;
    return t;
  }
  Tok str() {
    Tok t;
    t.pos = here();
    t.k = tStr;
    adv();
    while (!end() && c() != '"') {
      if (c() == '\n') fail("lex", t.pos, "unterminated string literal");
      if (c() == '\\') t.sval += escape(t.pos);
      else {
        t.sval += c();
        adv();
      }
    }
    if (end()) fail("lex", t.pos, "unterminated string literal");
    adv();
    return t;
  }
  Tok punct() {
    Tok t;
    t.pos = here();
    struct P { const char* s; T k; };
    static const P table[] = {
        {"<<=", pShlA}, {">>=", pShrA}, {"++", pInc}, {"--", pDec}, {"+=", pAddA},
        {"-=", pSubA}, {"->", pArrow}, {"*=", pMulA}, {"/=", pDivA}, {"%=", pRemA},
        {"&&", pAndAnd}, {"&=", pAndA}, {"||", pOrOr}, {"|=", pOrA}, {"^=", pXorA},
        {"!=", pNe}, {"==", pEq}, {"<<", pShl}, {">>", pShr}, {"<=", pLe}, {">=", pGe},
        {"(", pLP}, {")", pRP}, {"{", pLB}, {"}", pRB}, {"[", pLS}, {"]", pRS}, {";", pSemi},
        {",", pComma}, {"?", pQ}, {":", pColon}, {"~", pTilde}, {".", pDot}, {"+", pPlus},
        {"-", pMinus}, {"*", pStar}, {"/", pSlash}, {"%", pPct}, {"&", pAmp}, {"|", pPipe},
        {"^", pCaret}, {"!", pBang}, {"=", pAsg}, {"<", pLt}, {">", pGt}};
    for (const P& p : table) {
      size_t n = 0;
      while (p.s[n] && c(n) == p.s[n]) ++n;
      if (!p.s[n]) {
        for (size_t k = 0; k < n; ++k) adv();
        t.k = p.k;
        return t;
      }
    }
    fail("lex", t.pos, std::string("illegal character '") + c() + "'");
  }
  Tok any() {
    char ch = c();
    if (isalpha((unsigned char)ch) || ch == '_') return ident();
    if (isdigit((unsigned char)ch)) return number();
    if (ch == '\'') return chr();
    if (ch == '"') return str();
    return punct();
  }
};

// Blanks preprocessor lines in place (line numbers are preserved), keeping
// object-like #define replacements as token lists; #include lines vanish.
std::string preprocess(const std::string& src, std::map<std::string, std::vector<Tok>>& macros) {
  std::string out;
  out.reserve(src.size());
  int line = 1;
  size_t pos = 0;
  while (pos < src.size()) {
    size_t eol = src.find('\n', pos);
    if (eol == std::string::npos) eol = src.size();
    std::string text = src.substr(pos, eol - pos);
    size_t first = text.find_first_not_of(" \t");
    if (first != std::string::npos && text[first] == '#') {
      Pos at{line, (int)first + 1};
      std::string body = text.substr(first + 1);
      size_t b = body.find_first_not_of(" \t");
      std::string dir = b == std::string::npos ? std::string() : body.substr(b);
      if (dir.compare(0, 7, "include") == 0) {
        // dropped
      } else if (dir.compare(0, 6, "define") == 0) {
        std::string rest = dir.substr(6);
        size_t np = rest.find_first_not_of(" \t");
        if (np == std::string::npos) fail("lex", at, "#define without a name");
        size_t ne = np;
        while (ne < rest.size() && (isalnum((unsigned char)rest[ne]) || rest[ne] == '_')) ++ne;
        std::string name = rest.substr(np, ne - np);
        if (name.empty()) fail("lex", at, "#define without a name");
        if (ne < rest.size() && rest[ne] == '(')
          fail("lex", at, "function-like macro '" + name + "' is not supported");
        std::string value = rest.substr(ne);
        Scan sc(value);
        std::vector<Tok> repl;
        sc.skip();
        while (!sc.end()) {
          repl.push_back(sc.any());
          sc.skip();
        }
        macros[name] = std::move(repl);
      } else {
        fail("lex", at, "unsupported preprocessor directive");
      }
    } else {
      out += text;
    }
    if (eol < src.size()) out += '\n';
    pos = eol + 1;
    ++line;
  }
  return out;
}

std::vector<Tok> tokenize(const std::string& src) {
  std::map<std::string, std::vector<Tok>> macros;
  std::string text = preprocess(src, macros);
  Scan sc(text);
  std::vector<Tok> out;
  int launch = 0;
  struct Pend { Tok t; int depth; };
  std::vector<Pend> pend;
  while (true) {
    Tok t;
    int depth = 0;
    if (!pend.empty()) {
      t = pend.back().t;
      depth = pend.back().depth;
      pend.pop_back();
    } else {
      sc.skip();
      if (sc.end()) break;
      bool prevIdent = !out.empty() && out.back().k == tId;
      if (sc.c() == '<' && sc.c(1) == '<' && sc.c(2) == '<' && prevIdent && launch == 0) {
        t.k = pLaunchOpen;
        t.pos = sc.here();
        sc.adv(); sc.adv(); sc.adv();
      } else if (sc.c() == '>' && sc.c(1) == '>' && sc.c(2) == '>' && launch > 0) {
        t.k = pLaunchClose;
        t.pos = sc.here();
        sc.adv(); sc.adv(); sc.adv();
      } else {
        t = sc.any();
      }
    }
    if (t.k == tId) {
      auto it = macros.find(t.text);
      if (it != macros.end()) {
        if (depth + 1 > 32) fail("lex", t.pos, "macro expansion too deep");
        for (auto r = it->second.rbegin(); r != it->second.rend(); ++r) {
          Tok x = *r;
          x.pos = t.pos;  // diagnostics point at the use site
          pend.push_back(Pend{x, depth + 1});
        }
        continue;
      }
    }
    if (t.k == pLaunchOpen) ++launch;
    if (t.k == pLaunchClose) --launch;
    out.push_back(t);
  }
  Tok e;
  e.k = tEnd;
  e.pos = sc.here();
  out.push_back(e);
  return out;
}

struct Alias { int base; int ptr; };
const std::map<std::string, Alias>& aliases() {
  static const std::map<std::string, Alias> m = {
      {"cudaStream_t", {MCK_LONG, 0}}, {"cudaEvent_t", {MCK_LONG, 0}},
      {"cudaError_t", {MCK_INT, 0}}, {"size_t", {MCK_LONG, 0}}};
  return m;
}

class Parser {
 public:
  Parser(std::vector<Tok> toks, std::shared_ptr<Unit> u) : tk_(std::move(toks)), u_(std::move(u)) {}

  void run() {
    while (!is(tEnd)) topLevel();
  }

 private:
  std::vector<Tok> tk_;
  size_t p_ = 0;
  std::shared_ptr<Unit> u_;

  const Tok& cur() const { return tk_[p_]; }
  const Tok& ahead(size_t n) const { return p_ + n < tk_.size() ? tk_[p_ + n] : tk_.back(); }
  bool is(T k) const { return cur().k == k; }
  Tok take() { return tk_[p_++]; }
  bool accept(T k) {
    if (!is(k)) return false;
    ++p_;
    return true;
  }
  [[noreturn]] void expected(const std::string& what) {
    std::string found = cur().k == tId ? "'" + cur().text + "'" : tokDesc(cur().k);
    fail("parse", cur().pos, "expected " + what + ", found " + found);
  }
  Tok expect(T k, const std::string& what) {
    if (!is(k)) expected(what);
    return take();
  }

  bool isType(const Tok& t) const {
    switch (t.k) {
      case kVoid: case kChar: case kInt: case kUnsigned: case kLong: case kFloat: case kDouble:
        return true;
      case tId: return aliases().count(t.text) > 0;
      default: return false;
    }
  }

  Ty baseType() {
    Ty t;
    switch (cur().k) {
      case kVoid: t.base = MCK_VOID; take(); break;
      case kChar: t.base = MCK_CHAR; take(); break;
      case kInt: t.base = MCK_INT; take(); break;
      case kLong: t.base = MCK_LONG; take(); accept(kInt); break;
      case kFloat: t.base = MCK_FLOAT; take(); break;
      case kDouble: t.base = MCK_DOUBLE; take(); break;
      case kUnsigned: take(); accept(kInt); t.base = MCK_UINT; break;
      case tId: {
        auto it = aliases().find(cur().text);
        if (it == aliases().end()) expected("a type name");
        t.base = it->second.base;
        t.ptr = it->second.ptr;
        take();
        break;
      }
      default: expected("a type name");
    }
    return t;
  }

  // ---- expressions (precedence climbing; same table as parser.cpp:142-161) ----
  Expr* expr() { return assign(); }

  Expr* assign() {
    Expr* lhs = ternary();
    static const struct { T t; int op; } comp[] = {
        {pAddA, MCK_ADD}, {pSubA, MCK_SUB}, {pMulA, MCK_MUL}, {pDivA, MCK_DIV}, {pRemA, MCK_REM},
        {pShlA, MCK_SHL}, {pShrA, MCK_SHR}, {pAndA, MCK_BAND}, {pOrA, MCK_BOR}, {pXorA, MCK_BXOR}};
    if (is(pAsg)) {
      Expr* e = u_->newE(EK::Asg, take().pos);
      e->a = lhs;
      e->b = assign();
      return e;
    }
    for (const auto& c : comp)
      if (is(c.t)) {
        Expr* e = u_->newE(EK::Asg, take().pos);
        e->compound = true;
        e->op = c.op;
        e->a = lhs;
        e->b = assign();
        return e;
      }
    return lhs;
  }

  Expr* ternary() {
    Expr* c = binary(1);
    if (!is(pQ)) return c;
    Expr* e = u_->newE(EK::Cond, take().pos);
    e->a = c;
    e->b = assign();
    expect(pColon, "':'");
    e->c = assign();
    return e;
  }

  static bool binOp(T t, int& prec, int& op) {
    switch (t) {
      case pStar: prec = 10; op = MCK_MUL; return true;
      case pSlash: prec = 10; op = MCK_DIV; return true;
      case pPct: prec = 10; op = MCK_REM; return true;
      case pPlus: prec = 9; op = MCK_ADD; return true;
      case pMinus: prec = 9; op = MCK_SUB; return true;
      case pShl: prec = 8; op = MCK_SHL; return true;
      case pShr: prec = 8; op = MCK_SHR; return true;
      case pLt: prec = 7; op = MCK_LT; return true;
      case pLe: prec = 7; op = MCK_LE; return true;
      case pGt: prec = 7; op = MCK_GT; return true;
      case pGe: prec = 7; op = MCK_GE; return true;
      case pEq: prec = 6; op = MCK_EQ; return true;
      case pNe: prec = 6; op = MCK_NE; return true;
      case pAmp: prec = 5; op = MCK_BAND; return true;
      case pCaret: prec = 4; op = MCK_BXOR; return true;
      case pPipe: prec = 3; op = MCK_BOR; return true;
      case pAndAnd: prec = 2; op = MCK_LAND; return true;
      case pOrOr: prec = 1; op = MCK_LOR; return true;
      default: return false;
    }
  }

  Expr* binary(int minPrec) {
    Expr* lhs = unary();
    while (true) {
      int prec, op;
      if (!binOp(cur().k, prec, op) || prec < minPrec) return lhs;
      Pos at = take().pos;
      Expr* rhs = binary(prec + 1);
      Expr* e = u_->newE(EK::Bin, at);
      e->op = op;
      e->a = lhs;
      e->b = rhs;
      lhs = e;
    }
  }

  Expr* unaryNode(int op) {
    Expr* e = u_->newE(EK::Un, take().pos);
    e->op = op;
    e->a = unary();
    return e;
  }

  // unary operators beyond MCK_NEG/NOT/BITNOT
  static constexpr int kDeref = 10, kAddr = 11;

  Expr* unary() {
    Pos at = cur().pos;
    switch (cur().k) {
      case pInc:
      case pDec: {
        int d = cur().k == pInc ? 1 : -1;
        take();
        Expr* e = u_->newE(EK::IncDec, at);
        e->prefix = true;
        e->delta = d;
        e->a = unary();
        return e;
      }
      case pPlus: take(); return unary();
      case pMinus: return unaryNode(MCK_NEG);
      case pBang: return unaryNode(MCK_NOT);
      case pTilde: return unaryNode(MCK_BITNOT);
      case pStar: return unaryNode(kDeref);
      case pAmp: return unaryNode(kAddr);
      case kSizeof: {
        take();
        if (is(pLP) && isType(ahead(1))) {
          take();
          Ty t = baseType();
          while (accept(pStar)) ++t.ptr;
          expect(pRP, "')'");
          Expr* e = u_->newE(EK::Sizeof, at);
          e->castTy = t;
          return e;
        }
        Expr* operand = unary();
        Expr* e = u_->newE(EK::Sizeof, at);
        e->a = operand;
        return e;
      }
      case pLP:
        if (isType(ahead(1))) {
          take();
          Ty t = baseType();
          while (accept(pStar)) ++t.ptr;
          expect(pRP, "')'");
          Expr* e = u_->newE(EK::Cast, at);
          e->castTy = t;
          e->a = unary();
          return e;
        }
        return postfix(primary());
      default:
        return postfix(primary());
    }
  }

  Expr* primary() {
    Pos at = cur().pos;
    switch (cur().k) {
      case tInt: {
        Tok t = take();
        Expr* e = u_->newE(EK::Int, at);
        e->ival = t.ival;
        e->lit.base = t.isU ? MCK_UINT : t.isL ? MCK_LONG : MCK_INT;
        return e;
      }
      case tChr: {
        Tok t = take();
        Expr* e = u_->newE(EK::Int, at);
        e->ival = t.ival;
        e->lit.base = MCK_INT;
        return e;
      }
      case tFlt: {
        Tok t = take();
        Expr* e = u_->newE(EK::Flt, at);
        e->fval = t.fval;
        e->lit.base = t.isF ? MCK_FLOAT : MCK_DOUBLE;
        return e;
      }
      case tStr: {
        Tok t = take();
        Expr* e = u_->newE(EK::Str, at);
        e->sval = t.sval;
        return e;
      }
      case tId: {
        Tok t = take();
        Expr* e = u_->newE(EK::Name, at);
        e->text = t.text;
        return e;
      }
      case pLP: {
        take();
        Expr* e = expr();
        expect(pRP, "')'");
        return e;
      }
      default: expected("an expression");
    }
  }

  void argList(std::vector<Expr*>& out) {
    if (!is(pRP)) {
      out.push_back(assign());
      while (accept(pComma)) out.push_back(assign());
    }
    expect(pRP, "')'");
  }

  Expr* postfix(Expr* e) {
    while (true) {
      Pos at = cur().pos;
      if (accept(pLP)) {
        Expr* c = u_->newE(EK::Call, at);
        c->a = e;
        argList(c->args);
        e = c;
      } else if (accept(pLS)) {
        Expr* x = u_->newE(EK::Idx, at);
        x->a = e;
        x->b = expr();
        expect(pRS, "']'");
        e = x;
      } else if (accept(pDot)) {
        Tok name = expect(tId, "a member name");
        Expr* m = u_->newE(EK::Mem, at);
        m->a = e;
        m->text = name.text;
        e = m;
      } else if (is(pInc) || is(pDec)) {
        int d = is(pInc) ? 1 : -1;
        take();
        Expr* x = u_->newE(EK::IncDec, at);
        x->delta = d;
        x->a = e;
        e = x;
      } else if (accept(pLaunchOpen)) {
        Expr* l = u_->newE(EK::Launch, at);
        l->a = e;
        l->grid = assign();
        expect(pComma, "','");
        l->block = assign();
        if (accept(pComma)) {
          l->shmem = assign();
          if (accept(pComma)) l->stream = assign();
        }
        expect(pLaunchClose, "'>>>'");
        expect(pLP, "'('");
        argList(l->args);
        e = l;
      } else {
        return e;
      }
    }
  }

  // ---- statements ----
  bool atDecl() const { return is(kExtern) || is(kShared) || isType(cur()); }

  int64_t fold(const Expr* e) {
    switch (e->k) {
      case EK::Int: return e->ival;
      case EK::Sizeof:
        if (!e->a) return e->castTy.bytes();
        break;
      case EK::Un:
        if (e->op == MCK_NEG) return -fold(e->a);
        if (e->op == MCK_BITNOT) return ~fold(e->a);
        if (e->op == MCK_NOT) return !fold(e->a);
        break;
      case EK::Bin: {
        int64_t l = fold(e->a), r = fold(e->b);
        switch (e->op) {
          case MCK_ADD: return l + r;
          case MCK_SUB: return l - r;
          case MCK_MUL: return l * r;
          case MCK_DIV:
            if (!r) fail("parse", e->pos, "expected a nonzero divisor, found 0");
            return l / r;
          case MCK_REM:
            if (!r) fail("parse", e->pos, "expected a nonzero divisor, found 0");
            return l % r;
          case MCK_SHL: return l << r;
          case MCK_SHR: return l >> r;
          case MCK_BAND: return l & r;
          case MCK_BOR: return l | r;
          case MCK_BXOR: return l ^ r;
          default: break;
        }
        break;
      }
      default: break;
    }
    fail("parse", e->pos, "expected a constant expression, found a non-constant expression");
  }

  Declarator declarator(Ty base) {
    Declarator d;
    d.ty = base;
    while (accept(pStar)) ++d.ty.ptr;
    Tok n = expect(tId, "a declarator name");
    d.name = n.text;
    d.pos = n.pos;
    if (accept(pLS)) {
      if (is(pRS)) {
        d.ty.arr = 0;
      } else {
        Expr* len = expr();
        int64_t v = fold(len);
        if (v <= 0) fail("parse", len->pos, "expected a positive array length, found " + std::to_string(v));
        d.ty.arr = v;
      }
      expect(pRS, "']'");
      if (is(pLS)) expected("a 1-D array (multi-dimensional arrays are not supported)");
    }
    if (accept(pAsg)) d.init = assign();
    return d;
  }

  Stmt* declStmt() {
    Pos at = cur().pos;
    bool ext = accept(kExtern);
    bool sh = accept(kShared);
    if (sh && !ext)
      fail("parse", at, "expected 'extern __shared__' (static __shared__ is not supported), found '__shared__'");
    if (ext && !sh) expected("'__shared__' after 'extern'");
    Ty base = baseType();
    Stmt* s = u_->newS(SK::Decl, at);
    s->externShared = ext && sh;
    s->decls.push_back(declarator(base));
    while (accept(pComma)) s->decls.push_back(declarator(base));
    expect(pSemi, "';'");
    if (s->externShared)
      for (auto& d : s->decls) {
        if (!d.ty.isArray() || d.ty.arr != 0)
          fail("parse", d.pos, "expected an unsized array declarator for extern __shared__, found " + d.name);
        d.dynShared = true;
      }
    return s;
  }

  Stmt* stmt() {
    Pos at = cur().pos;
    switch (cur().k) {
      case pLB: return block();
      case kIf: {
        take();
        expect(pLP, "'('");
        Stmt* s = u_->newS(SK::If, at);
        s->cond = expr();
        expect(pRP, "')'");
        s->thenS = stmt();
        if (accept(kElse)) s->elseS = stmt();
        return s;
      }
      case kWhile: {
        take();
        expect(pLP, "'('");
        Stmt* s = u_->newS(SK::While, at);
        s->cond = expr();
        expect(pRP, "')'");
        s->loop = stmt();
        return s;
      }
      case kFor: {
        take();
        expect(pLP, "'('");
        Stmt* s = u_->newS(SK::For, at);
        if (is(pSemi)) {
          s->init = u_->newS(SK::Empty, cur().pos);
          take();
        } else if (atDecl()) {
          s->init = declStmt();
        } else {
          Stmt* i = u_->newS(SK::ExprS, cur().pos);
          i->e = expr();
          s->init = i;
          expect(pSemi, "';'");
        }
        if (!is(pSemi)) s->cond = expr();
        expect(pSemi, "';'");
        if (!is(pRP)) s->incr = expr();
        expect(pRP, "')'");
        s->loop = stmt();
        return s;
      }
      case kReturn: {
        take();
        Stmt* s = u_->newS(SK::Ret, at);
        if (!is(pSemi)) s->e = expr();
        expect(pSemi, "';'");
        return s;
      }
      case kBreak:
        take();
        expect(pSemi, "';'");
        return u_->newS(SK::Brk, at);
      case kContinue:
        take();
        expect(pSemi, "';'");
        return u_->newS(SK::Cont, at);
      case pSemi:
        take();
        return u_->newS(SK::Empty, at);
      default: {
        if (atDecl()) return declStmt();
        Stmt* s = u_->newS(SK::ExprS, at);
        s->e = expr();
        expect(pSemi, "';'");
        return s;
      }
    }
  }

  Stmt* block() {
    Pos at = expect(pLB, "'{'").pos;
    Stmt* s = u_->newS(SK::Block, at);
    while (!is(pRB)) {
      if (is(tEnd)) expected("'}'");
      s->body.push_back(stmt());
    }
    take();
    return s;
  }

  void topLevel() {
    Pos at = cur().pos;
    bool g = false, d = false, h = false;
    while (true) {
      if (accept(kGlobal)) {
        if (g) fail("parse", at, "expected at most one '__global__', found '__global__'");
        g = true;
      } else if (accept(kDevice)) {
        if (d) fail("parse", at, "expected at most one '__device__', found '__device__'");
        d = true;
      } else if (accept(kHost)) {
        if (h) fail("parse", at, "expected at most one '__host__', found '__host__'");
        h = true;
      } else if (accept(kNoinline) || accept(kForceinline)) {
      } else {
        break;
      }
    }
    Ty base = baseType();
    Ty ty = base;
    while (accept(pStar)) ++ty.ptr;
    Tok name = expect(tId, "a declaration name");
    if (accept(pLP)) {
      Function f;
      f.name = name.text;
      f.ret = ty;
      f.pos = at;
      if (g && (d || h))
        fail("parse", at, "expected '__global__' without other execution-space attributes, found conflicting attributes");
      f.space = g ? 3 : (d && h) ? 2 : d ? 1 : 0;
      if (is(kVoid) && ahead(1).k == pRP) {
        take();
        take();
      } else if (!accept(pRP)) {
        while (true) {
          Param p;
          p.ty = baseType();
          while (accept(pStar)) ++p.ty.ptr;
          p.pos = cur().pos;
          if (is(tId)) p.name = take().text;
          if (accept(pLS)) {
            if (!is(pRS)) expr();
            expect(pRS, "']'");
            ++p.ty.ptr;
          }
          f.params.push_back(p);
          if (!accept(pComma)) break;
        }
        expect(pRP, "')'");
      }
      if (!accept(pSemi)) {
        for (const auto& p : f.params)
          if (p.name.empty())
            fail("parse", p.pos, "expected a named parameter in a function definition, found an unnamed parameter");
        f.body = block();
      }
      u_->fns.push_back(std::move(f));
      return;
    }
    if (g || h) fail("parse", at, "expected a function after '__global__'/'__host__', found a variable");
    GlobalDef gd;
    gd.name = name.text;
    gd.ty = ty;
    gd.device = d;
    gd.pos = at;
    if (accept(pLS)) {
      if (is(pRS)) fail("parse", cur().pos, "expected an array length, found ']'");
      Expr* len = expr();
      gd.ty.arr = fold(len);
      if (gd.ty.arr <= 0) fail("parse", at, "expected a positive array length, found " + std::to_string(gd.ty.arr));
      expect(pRS, "']'");
    }
    if (accept(pAsg)) gd.init = assign();
    u_->globals.push_back(gd);
    while (accept(pComma)) {
      GlobalDef g2;
      g2.ty = base;
      while (accept(pStar)) ++g2.ty.ptr;
      Tok n2 = expect(tId, "a declaration name");
      g2.name = n2.text;
      g2.device = d;
      g2.pos = n2.pos;
      if (accept(pAsg)) g2.init = assign();
      u_->globals.push_back(g2);
    }
    expect(pSemi, "';'");
  }
};

}  // namespace

std::shared_ptr<Unit> parseUnit(const std::string& source, const std::string& filename) {
  auto u = std::make_shared<Unit>();
  u->filename = filename;
  Parser p(tokenize(source), u);
  p.run();
  return u;
}

}  // namespace mckb
