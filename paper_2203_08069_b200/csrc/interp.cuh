// Program format of the exact-order nest evaluator (td_nest_eval).
// Mirrored byte for byte by paper_2203_08069_b200/interp.py (ctypes).
#pragma once
#include <cstdint>

#define TD_MAX_LOOPS 16
#define TD_MAX_VARS 48
#define TD_MAX_ACC 8
#define TD_MAX_DIMS 8
#define TD_MAX_CODE 64
#define TD_MAX_OVER 4

// variable slots are evaluated in slot order; slot values are int64
enum { TD_VAR_LOOP = 0, TD_VAR_STRIP = 1, TD_VAR_ROTATE = 2 };
// postfix expression ops
enum { TD_OP_CONST = 0, TD_OP_LOAD = 1, TD_OP_ADD = 2, TD_OP_MUL = 3 };

struct td_var_def {
  int32_t kind;       // TD_VAR_*
  int32_t a;          // LOOP: loop index; STRIP: outer slot; ROTATE: result slot
  int32_t b;          // STRIP: inner slot
  int32_t nover;      // ROTATE: number of offset slots
  int32_t over[TD_MAX_OVER];
  int64_t block;      // STRIP: block size
  int64_t extent;     // STRIP: guard extent; ROTATE: modulus
};

struct td_access {
  const double* base;          // element at coordinate `origin`
  int32_t ndim;
  int32_t pad;
  int32_t slot[TD_MAX_DIMS];   // variable slot per axis
  int64_t origin[TD_MAX_DIMS];
  int64_t stride[TD_MAX_DIMS];
};

struct td_nest_prog {
  int32_t nloops, nvars, nacc, ncode;
  int32_t reduce;      // 1: out (+)= per point, 0: out = value
  int32_t serial;      // 1: one thread walks the whole nest
  int32_t npar;        // number of parallel (output-determining) loops
  int32_t pad;
  int64_t lo[TD_MAX_LOOPS];
  int64_t hi[TD_MAX_LOOPS];
  int32_t par[TD_MAX_LOOPS];   // loop indices of the parallel loops, nest order
  td_var_def vars[TD_MAX_VARS];
  td_access out;
  td_access acc[TD_MAX_ACC];
  int32_t op[TD_MAX_CODE];
  int32_t arg[TD_MAX_CODE];
  double konst[TD_MAX_CODE];
};
