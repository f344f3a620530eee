// program.hpp -- a lowered program: the step-exact IR (include/mck_ir.h) plus
// the symbol tables the host and device interpreters need.  Built once by
// compileProgram() (lower.cpp), immutable afterwards, shared by value.
#pragma once
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "ast.hpp"
#include "mck_ir.h"

namespace mckb {

struct GlobalInfo {
  std::string name;
  uint8_t type = 0;
  int64_t size = 0;
  bool device = false;
  bool hasInit = false;
  int64_t ival = 0;
  double fval = 0;
};

struct Program {
  std::shared_ptr<Unit> unit;
  std::string filename;
  std::vector<mck_ins> code;
  std::vector<mck_fn> fns;
  std::vector<mck_local> locals;
  std::vector<std::string> strings;  // names, printf formats
  std::vector<std::string> fnNames;
  std::vector<GlobalInfo> globals;
  int mainIndex = -1;
  int sharedDefaultName = -1;  // "(dynamic shared)" (device.cpp:33-38)

  int intern(const std::string& s);
  const std::string& str(int id) const { return strings[static_cast<size_t>(id)]; }
  std::string disassemble() const;

 private:
  std::map<std::string, int> ids_;
};

// lex + parse + lower + IR codegen; throws FrontendFailure.
std::shared_ptr<const Program> compileProgram(const std::string& source, const std::string& filename);

}  // namespace mckb
