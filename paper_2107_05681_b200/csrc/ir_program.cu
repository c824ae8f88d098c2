// ir_program.cu — reader and lowering of the reference's textual mini-IR for
// the GPU warp interpreter (host code).  Grammar: SPEC.md:111-121 /
// proj/README.md:37-67; opcode names proj/src/ir.cpp:17-46; operand forms per
// opcode as the reference parser accepts them (proj/src/parser.cpp:249-420:
// a shared access may omit the array name when the function declares exactly
// one shared array; `const` takes an immediate; phis need >= 2 incomings).
#include <algorithm>
#include <cctype>
#include <map>
#include <stdexcept>

#include "ir_program.h"

namespace darm_gpu {

namespace {

const char *const kOpNames[kNumOps] = {
    "add", "sub", "mul", "div", "rem", "and", "or", "xor", "shl", "shr",
    "icmp.eq", "icmp.ne", "icmp.lt", "icmp.gt", "icmp.le", "icmp.ge",
    "select", "load.shared", "store.shared", "load.global", "store.global",
    "tid", "const", "phi", "br", "condbr", "ret", "barrier"};

struct Tok {
  enum Kind { Value, Label, Int, Ident, Undef, Punct, Newline, End } kind = End;
  std::string text;
  int64_t value = 0;
  int line = 0;
};

class Lexer {
 public:
  explicit Lexer(const std::string &s) : s_(s) {}
  Tok next() {
    while (pos_ < s_.size()) {
      const char c = s_[pos_];
      if (c == '#') {
        while (pos_ < s_.size() && s_[pos_] != '\n') ++pos_;
      } else if (c == ' ' || c == '\t' || c == '\r') {
        ++pos_;
      } else {
        break;
      }
    }
    Tok t;
    t.line = line_;
    if (pos_ >= s_.size()) return t;
    const char c = s_[pos_];
    if (c == '\n') {
      ++pos_;
      ++line_;
      t.kind = Tok::Newline;
      return t;
    }
    if (c == '%' || c == '^') {
      ++pos_;
      t.text = name();
      if (t.text.empty()) fail(t.line, "expected a name");
      t.kind = c == '%' ? Tok::Value : Tok::Label;
      return t;
    }
    if (std::isdigit((unsigned char)c) || (c == '-' && pos_ + 1 < s_.size() && std::isdigit((unsigned char)s_[pos_ + 1]))) {
      std::string num(1, c);
      ++pos_;
      while (pos_ < s_.size() && std::isdigit((unsigned char)s_[pos_])) num.push_back(s_[pos_++]);
      t.kind = Tok::Int;
      try {
        t.value = std::stoll(num);
      } catch (...) {
        fail(t.line, "integer out of range");
      }
      return t;
    }
    if (std::isalpha((unsigned char)c) || c == '_' || c == '.') {
      t.text = name();
      t.kind = t.text == "undef" ? Tok::Undef : Tok::Ident;
      return t;
    }
    if (std::string("(){}[]:,=").find(c) != std::string::npos) {
      ++pos_;
      t.kind = Tok::Punct;
      t.text = std::string(1, c);
      return t;
    }
    fail(t.line, std::string("unexpected character '") + c + "'");
    return t;
  }
  [[noreturn]] static void fail(int line, const std::string &msg) {
    throw std::runtime_error("line " + std::to_string(line) + ": " + msg);
  }

 private:
  std::string name() {
    std::string n;
    while (pos_ < s_.size() && (std::isalnum((unsigned char)s_[pos_]) || s_[pos_] == '_' || s_[pos_] == '.'))
      n.push_back(s_[pos_++]);
    return n;
  }
  const std::string &s_;
  size_t pos_ = 0;
  int line_ = 1;
};

struct RawOperand {
  enum Kind { None, Value, Imm, Undef, Label, Mem } kind = None;
  std::string text;
  int32_t imm = 0;
};

struct RawInst {
  int op = -1;
  std::string result;
  std::vector<RawOperand> ops;                                   // data / label / mem operands
  std::vector<std::pair<RawOperand, std::string>> incomings;     // phi
  int line = 0;
};

struct RawBlock {
  std::string name;
  std::vector<RawInst> phis, body;
  RawInst term;
};

class Parser {
 public:
  explicit Parser(const std::string &text) : lex_(text) { bump(); }

  void parse(std::vector<std::pair<std::string, int64_t>> &globals, std::string &fname,
             std::vector<std::string> &params, std::vector<std::pair<std::string, int64_t>> &shared,
             std::vector<RawBlock> &blocks) {
    skip_nl();
    bool have_fn = false;
    while (cur_.kind != Tok::End) {
      if (cur_.kind == Tok::Ident && cur_.text == "global") {
        bump();
        const std::string n = ident("global name");
        globals.push_back({n, bracket_size()});
      } else if (cur_.kind == Tok::Ident && cur_.text == "fn") {
        if (have_fn) {   // only the first function is lowered; skip the rest
          while (cur_.kind != Tok::End && !(cur_.kind == Tok::Punct && cur_.text == "}")) bump();
          if (cur_.kind != Tok::End) bump();
        } else {
          have_fn = true;
          parse_fn(fname, params, shared, blocks);
        }
      } else {
        Lexer::fail(cur_.line, "expected 'global' or 'fn'");
      }
      skip_nl();
    }
    if (!have_fn) throw std::runtime_error("no function in module");
  }

 private:
  void bump() { cur_ = lex_.next(); }
  void skip_nl() {
    while (cur_.kind == Tok::Newline) bump();
  }
  bool at(const char *p) const { return cur_.kind == Tok::Punct && cur_.text == p; }
  void expect(const char *p) {
    if (!at(p)) Lexer::fail(cur_.line, std::string("expected '") + p + "'");
    bump();
  }
  std::string ident(const char *what) {
    if (cur_.kind != Tok::Ident) Lexer::fail(cur_.line, std::string("expected ") + what);
    std::string s = cur_.text;
    bump();
    return s;
  }
  int64_t bracket_size() {
    expect("[");
    if (cur_.kind != Tok::Int || cur_.value < 0) Lexer::fail(cur_.line, "expected a size");
    const int64_t v = cur_.value;
    bump();
    expect("]");
    return v;
  }
  RawOperand value_or_imm() {
    RawOperand o;
    if (cur_.kind == Tok::Value) {
      o.kind = RawOperand::Value;
      o.text = cur_.text;
    } else if (cur_.kind == Tok::Int) {
      if (cur_.value < INT32_MIN || cur_.value > INT32_MAX) Lexer::fail(cur_.line, "immediate out of 32-bit range");
      o.kind = RawOperand::Imm;
      o.imm = int32_t(cur_.value);
    } else if (cur_.kind == Tok::Undef) {
      o.kind = RawOperand::Undef;
    } else {
      Lexer::fail(cur_.line, "expected value or immediate");
    }
    bump();
    return o;
  }
  std::string label() {
    if (cur_.kind != Tok::Label) Lexer::fail(cur_.line, "expected ^label");
    std::string s = cur_.text;
    bump();
    return s;
  }
  RawOperand mem_name(bool shared, size_t n_shared, const std::string &only_shared) {
    RawOperand o;
    o.kind = RawOperand::Mem;
    if (cur_.kind == Tok::Ident) {
      o.text = cur_.text;
      bump();
      return o;
    }
    if (shared && n_shared == 1) {
      o.text = only_shared;
      return o;
    }
    Lexer::fail(cur_.line, shared ? "shared access needs an array name" : "expected memory name");
  }

  void parse_fn(std::string &fname, std::vector<std::string> &params,
                std::vector<std::pair<std::string, int64_t>> &shared, std::vector<RawBlock> &blocks) {
    bump();   // fn
    fname = ident("function name");
    expect("(");
    while (!at(")")) {
      if (cur_.kind != Tok::Value) Lexer::fail(cur_.line, "expected %param");
      params.push_back(cur_.text);
      bump();
      if (at(",")) bump();
    }
    expect(")");
    while (cur_.kind == Tok::Ident && cur_.text == "shared") {
      bump();
      const std::string n = ident("shared array name");
      shared.push_back({n, bracket_size()});
    }
    expect("{");
    skip_nl();
    while (!at("}")) {
      if (cur_.kind != Tok::Label) Lexer::fail(cur_.line, "expected block label");
      RawBlock b;
      b.name = cur_.text;
      for (const auto &o : blocks)
        if (o.name == b.name) Lexer::fail(cur_.line, "duplicate block '^" + b.name + "'");
      bump();
      expect(":");
      skip_nl();
      bool done = false;
      while (!done) {
        if (at("}") || cur_.kind == Tok::End) Lexer::fail(cur_.line, "block '^" + b.name + "' has no terminator");
        RawInst in;
        in.line = cur_.line;
        if (cur_.kind == Tok::Value) {
          in.result = cur_.text;
          bump();
          expect("=");
        }
        if (cur_.kind != Tok::Ident) Lexer::fail(cur_.line, "expected opcode");
        for (int k = 0; k < kNumOps; ++k)
          if (cur_.text == kOpNames[k]) in.op = k;
        if (in.op < 0) Lexer::fail(cur_.line, "unknown opcode '" + cur_.text + "'");
        bump();
        const bool has_result = !(in.op == kStoreShared || in.op == kStoreGlobal || in.op == kBr ||
                                  in.op == kCondBr || in.op == kRet || in.op == kBarrier);
        if (has_result && in.result.empty()) Lexer::fail(in.line, std::string(kOpNames[in.op]) + " needs a result");
        if (!has_result && !in.result.empty()) Lexer::fail(in.line, std::string(kOpNames[in.op]) + " has no result");
        const std::string only = shared.size() == 1 ? shared[0].first : std::string();
        switch (in.op) {
          case kPhi:
            while (true) {
              RawOperand v = value_or_imm();
              expect(":");
              in.incomings.push_back({v, label()});
              if (at(","))
                bump();
              else
                break;
            }
            if (in.incomings.size() < 2) Lexer::fail(in.line, "phi needs at least two incomings");
            if (!b.body.empty()) Lexer::fail(in.line, "phi after non-phi");
            break;
          case kSelect:
            for (int k = 0; k < 3; ++k) in.ops.push_back(value_or_imm());
            break;
          case kLoadShared:
          case kLoadGlobal:
            in.ops.push_back(mem_name(in.op == kLoadShared, shared.size(), only));
            in.ops.push_back(value_or_imm());
            break;
          case kStoreShared:
          case kStoreGlobal:
            in.ops.push_back(mem_name(in.op == kStoreShared, shared.size(), only));
            in.ops.push_back(value_or_imm());
            in.ops.push_back(value_or_imm());
            break;
          case kTid:
          case kBarrier:
            break;
          case kConst:
            in.ops.push_back(value_or_imm());
            if (in.ops[0].kind == RawOperand::Value) Lexer::fail(in.line, "const takes an immediate");
            break;
          case kBr: {
            RawOperand l;
            l.kind = RawOperand::Label;
            l.text = label();
            in.ops.push_back(l);
            break;
          }
          case kCondBr: {
            in.ops.push_back(value_or_imm());
            for (int k = 0; k < 2; ++k) {
              RawOperand l;
              l.kind = RawOperand::Label;
              l.text = label();
              in.ops.push_back(l);
            }
            break;
          }
          case kRet:
            if (cur_.kind == Tok::Value || cur_.kind == Tok::Int || cur_.kind == Tok::Undef)
              in.ops.push_back(value_or_imm());
            break;
          default:   // the binary ALU / compare opcodes
            in.ops.push_back(value_or_imm());
            in.ops.push_back(value_or_imm());
            break;
        }
        if (cur_.kind != Tok::Newline && !at("}")) Lexer::fail(cur_.line, "unexpected token after instruction");
        skip_nl();
        if (in.op == kBr || in.op == kCondBr || in.op == kRet) {
          b.term = in;
          done = true;
        } else if (in.op == kPhi) {
          b.phis.push_back(in);
        } else {
          b.body.push_back(in);
        }
      }
      blocks.push_back(std::move(b));
    }
    expect("}");
  }

  Lexer lex_;
  Tok cur_;
};

}  // namespace

void default_latencies(int64_t *lat) {
  for (int k = 0; k < kNumOps; ++k) lat[k] = 1;
  lat[kLoadShared] = lat[kStoreShared] = 20;
  lat[kLoadGlobal] = lat[kStoreGlobal] = 100;
}

IrProgram compile_ir(const std::string &text) {
  std::vector<std::pair<std::string, int64_t>> globals, shared;
  std::vector<RawBlock> raw;
  IrProgram P;
  Parser(text).parse(globals, P.name, P.params, shared, raw);
  if (raw.empty()) throw std::runtime_error("function '" + P.name + "' has no blocks");
  default_latencies(P.latency);

  // memories: globals (declaration order), then shared arrays
  for (const auto &g : globals) {
    P.mems.push_back({g.first, g.second, false, P.global_words});
    P.global_words += g.second;
  }
  for (const auto &s : shared) {
    P.mems.push_back({s.first, s.second, true, P.shared_words});
    P.shared_words += s.second;
  }
  P.n_globals = int(globals.size());
  P.n_shared = int(shared.size());
  if (P.mems.size() > 255) throw std::runtime_error("too many memories");

  // registers: params first, then every other %name in order of appearance
  std::map<std::string, int> reg;
  for (const auto &p : P.params) {
    if (reg.count(p)) throw std::runtime_error("duplicate parameter '%" + p + "'");
    reg[p] = int(reg.size());
    P.reg_names.push_back(p);
  }
  auto reg_of = [&](const std::string &n) {
    auto it = reg.find(n);
    if (it != reg.end()) return it->second;
    const int i = int(reg.size());
    reg[n] = i;
    P.reg_names.push_back(n);
    return i;
  };
  auto operand = [&](const RawOperand &o) {
    IrOperand r;
    if (o.kind == RawOperand::Value) {
      r.kind = kOpndReg;
      r.v = reg_of(o.text);
    } else if (o.kind == RawOperand::Imm) {
      r.kind = kOpndImm;
      r.v = o.imm;
    } else if (o.kind == RawOperand::Undef) {
      r.kind = kOpndUndef;
    }
    return r;
  };
  std::map<std::string, int> bidx;
  for (size_t b = 0; b < raw.size(); ++b) {
    bidx[raw[b].name] = int(b);
    P.block_names.push_back(raw[b].name);
  }
  auto block_of = [&](const std::string &n, int line) {
    auto it = bidx.find(n);
    if (it == bidx.end()) Lexer::fail(line, "branch to unknown block '^" + n + "'");
    return it->second;
  };
  auto mem_of = [&](const std::string &n, bool want_shared, int line) {
    for (size_t m = 0; m < P.mems.size(); ++m)
      if (P.mems[m].name == n && P.mems[m].shared == want_shared) return int(m);
    Lexer::fail(line, "unknown memory '" + n + "'");
  };
  for (const auto &rb : raw) {
    IrBlock B;
    B.first_phi = int(P.phis.size());
    B.n_phi = int(rb.phis.size());
    for (const auto &ph : rb.phis) {
      IrPhi p;
      p.dst = reg_of(ph.result);
      p.first = int(P.phi_ins.size());
      p.count = int(ph.incomings.size());
      for (const auto &in : ph.incomings) P.phi_ins.push_back({block_of(in.second, ph.line), operand(in.first)});
      P.phis.push_back(p);
    }
    B.first_inst = int(P.insts.size());
    B.n_inst = int(rb.body.size());
    for (const auto &ri : rb.body) {
      IrInst I;
      I.op = uint8_t(ri.op);
      I.dst = ri.result.empty() ? int16_t(-1) : int16_t(reg_of(ri.result));
      size_t k0 = 0;
      if (ri.op == kLoadShared || ri.op == kLoadGlobal || ri.op == kStoreShared || ri.op == kStoreGlobal) {
        I.mem = uint8_t(mem_of(ri.ops[0].text, ri.op == kLoadShared || ri.op == kStoreShared, ri.line));
        k0 = 1;
      }
      for (size_t k = k0; k < ri.ops.size(); ++k) I.a[k - k0] = operand(ri.ops[k]);
      P.insts.push_back(I);
    }
    B.term = uint8_t(rb.term.op);
    B.succ[0] = B.succ[1] = -1;
    if (rb.term.op == kBr) {
      B.succ[0] = block_of(rb.term.ops[0].text, rb.term.line);
    } else if (rb.term.op == kCondBr) {
      B.cond = operand(rb.term.ops[0]);
      B.succ[0] = block_of(rb.term.ops[1].text, rb.term.line);
      B.succ[1] = block_of(rb.term.ops[2].text, rb.term.line);
    } else {
      if (!rb.term.ops.empty()) B.cond = operand(rb.term.ops[0]);
      if (P.ret_block >= 0) throw std::runtime_error("function '" + P.name + "' has multiple ret blocks");
      P.ret_block = int(P.blocks.size());
    }
    B.ipdom = -1;
    P.blocks.push_back(B);
  }
  if (P.ret_block < 0) throw std::runtime_error("function '" + P.name + "' has no ret block");
  if (reg.size() > 32767) throw std::runtime_error("too many values");

  // immediate post-dominators on the reverse CFG rooted at the ret block
  // (iterative dataflow over bit sets; blocks that cannot reach ret get none)
  const int nb = int(P.blocks.size());
  const int words = (nb + 63) / 64;
  std::vector<std::vector<uint64_t>> pd(size_t(nb), std::vector<uint64_t>(size_t(words), ~uint64_t(0)));
  std::vector<bool> reach(size_t(nb), false);
  reach[size_t(P.ret_block)] = true;
  for (bool ch = true; ch;) {
    ch = false;
    for (int b = 0; b < nb; ++b)
      if (!reach[size_t(b)])
        for (int s : P.blocks[size_t(b)].succ)
          if (s >= 0 && reach[size_t(s)]) {
            reach[size_t(b)] = true;
            ch = true;
          }
  }
  for (int b = 0; b < nb; ++b)
    if (b == P.ret_block) {
      std::fill(pd[size_t(b)].begin(), pd[size_t(b)].end(), 0);
      pd[size_t(b)][size_t(b / 64)] |= uint64_t(1) << (b % 64);
    }
  for (bool ch = true; ch;) {
    ch = false;
    for (int b = 0; b < nb; ++b) {
      if (b == P.ret_block || !reach[size_t(b)]) continue;
      std::vector<uint64_t> x(size_t(words), ~uint64_t(0));
      for (int s : P.blocks[size_t(b)].succ)
        if (s >= 0 && reach[size_t(s)])
          for (int w = 0; w < words; ++w) x[size_t(w)] &= pd[size_t(s)][size_t(w)];
      x[size_t(b / 64)] |= uint64_t(1) << (b % 64);
      if (x != pd[size_t(b)]) {
        pd[size_t(b)] = x;
        ch = true;
      }
    }
  }
  auto count = [&](const std::vector<uint64_t> &v) {
    int c = 0;
    for (uint64_t w : v) c += __builtin_popcountll(w);
    return c;
  };
  for (int b = 0; b < nb; ++b) {
    if (!reach[size_t(b)] || b == P.ret_block) continue;
    const int want = count(pd[size_t(b)]) - 1;
    for (int c = 0; c < nb; ++c)
      if (c != b && (pd[size_t(b)][size_t(c / 64)] >> (c % 64) & 1) && reach[size_t(c)] && count(pd[size_t(c)]) == want)
        P.blocks[size_t(b)].ipdom = c;
  }
  return P;
}

}  // namespace darm_gpu
