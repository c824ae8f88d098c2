// ir_program.h — a mini-IR function compiled for the GPU warp interpreter
// (interp.cu): the textual IR of the reference (SPEC.md:111-121,
// proj/README.md:37-67) parsed by this library's own reader and lowered to
// flat arrays of instructions with integer operands, plus the immediate
// post-dominator of every block (the reconvergence points of
// interp.cpp:301-306).  Host code; not part of the public boundary.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace darm_gpu {

// Opcode numbering of the reference's enum (proj/include/darm/ir.hpp:17-46).
enum IrOp : uint8_t {
  kAdd, kSub, kMul, kDiv, kRem, kAnd, kOr, kXor, kShl, kShr,
  kIcmpEq, kIcmpNe, kIcmpLt, kIcmpGt, kIcmpLe, kIcmpGe,
  kSelect, kLoadShared, kStoreShared, kLoadGlobal, kStoreGlobal,
  kTid, kConst, kPhi, kBr, kCondBr, kRet, kBarrier,
  kNumOps
};

// operand kinds
enum : uint8_t { kOpndNone = 0, kOpndReg = 1, kOpndImm = 2, kOpndUndef = 3 };

struct IrOperand {
  uint8_t kind = kOpndNone;
  int32_t v = 0;          // register index or immediate
};

struct IrInst {            // 32 bytes
  uint8_t op = 0;
  uint8_t mem = 0;         // memory index (loads / stores)
  int16_t dst = -1;        // result register, -1 if none
  IrOperand a[3];          // data operands (loads: a[0] = index; stores: a[0] = index, a[1] = value)
};

struct IrPhiIn {
  int32_t pred;            // predecessor block index
  IrOperand val;
};

struct IrPhi {
  int32_t dst;
  int32_t first, count;    // range in phi_ins
};

struct IrBlock {
  int32_t first_inst, n_inst;   // body range in insts
  int32_t first_phi, n_phi;     // range in phis
  uint8_t term;                 // kBr / kCondBr / kRet
  IrOperand cond;               // condbr condition / ret value (kind None: void ret)
  int32_t succ[2];              // br: succ[0]; condbr: true, false
  int32_t ipdom;                // immediate post-dominator (-1: none)
};

struct IrMem {
  std::string name;
  int64_t size;
  bool shared;
  int64_t offset;          // word offset inside its class (globals / shared) of one warp
};

struct IrProgram {
  std::string name;
  std::vector<std::string> params;     // register i = param i
  std::vector<std::string> reg_names;  // every register
  std::vector<IrMem> mems;             // globals (declaration order), then shared arrays
  int n_globals = 0, n_shared = 0;
  int64_t global_words = 0, shared_words = 0;
  std::vector<IrBlock> blocks;
  std::vector<IrInst> insts;
  std::vector<IrPhi> phis;
  std::vector<IrPhiIn> phi_ins;
  std::vector<std::string> block_names;
  int entry = 0, ret_block = -1;
  int64_t latency[kNumOps];
};

// Parses the module text (first function) and lowers it; throws
// std::runtime_error with a line number on malformed input.
IrProgram compile_ir(const std::string &text);

// The reference's default latency model (proj/src/ir.cpp:235-244): every
// opcode 1 cycle, shared-memory accesses 20, global-memory accesses 100.
void default_latencies(int64_t *lat);

}  // namespace darm_gpu
