// Plain-old-data structures shared by the host plan builder (pt_plan.cpp)
// and the device executor (pt_exec.cu).
//
// A "program" is a DAG of tasks over interface vectors.  Every task writes
// a disjoint piece of one vector (rows of one m-block, or a slot range of a
// PLR t-buffer) and is computed entirely by one CTA in a fixed summation
// order, so results are bitwise repeatable no matter which CTA runs it
// (the reference pins bitwise-repeatable applies, test_solver.py:93-117).
// Dependencies are counters: a producer group of n tasks bumps its counter
// n times; consumers wait for the count.
#pragma once
#include <stdint.h>

namespace pt {

// vector slots of a program launch (base pointers supplied per launch)
enum Slot : int32_t {
  SLOT_IN = 0,    // program input vector (x, r, rhs ...)
  SLOT_OUT = 1,   // program output vector
  SLOT_Y = 2,     // A-apply result inside an A->M program
  SLOT_U1 = 3,    // sweep iterates
  SLOT_U2 = 4,
  SLOT_PRE = 5,   // pre-phase partial sums of the sweeps
  SLOT_T = 6,     // PLR t = Vt x buffers (one region per term instance)
  SLOT_AUX = 7,   // second input (u_in of gs_sweep)
  N_SLOTS = 8
};

enum TaskType : int32_t {
  TASK_Y_DENSE = 0,  // rows of an output block from dense kernel terms
  TASK_Y_PLR = 1,    // rows of an output block from PLR terms (U t)
  TASK_T_PLR = 2,    // t = Vt (sum of sources) for a slot range of a term
};

struct VecRef {
  int32_t slot;
  int32_t pad;
  int64_t off;  // complex-element offset into the slot vector
};

// one kernel term: scale * K (src0 [+ src1])
struct DevTerm {
  int32_t kernel;
  int32_t nsrc;
  double scale_re, scale_im;
  VecRef src[2];
  int64_t t_base;  // PLR: offset of this term instance's t in SLOT_T
};

// one identity term: coef * v
struct DevEye {
  double re, im;
  VecRef src;
};

struct DevWait {
  int32_t ctr;
  int32_t val;
};

// One contiguous operator range a task stages into a ring stage with a TMA
// bulk copy.  Y_PLR: whole rank columns [f0, f1) of the task's flat column
// list.  T_PLR: slots [f0, f1) of the task; e0 = its rows per consumer lane
// class, n32 | n16 << 10 | n8 << 20 (the piece's items are in class order).
// Y_DENSE: rows r0..r1 of term f0's kernel.
struct DevPiece {
  int64_t src;     // element offset into the operator pool (dense or factors)
  int32_t elems;
  int32_t f0, f1;
  int32_t e0;
  // Y_PLR: a second contiguous range that lands right behind the first in the
  // same stage (the next term's columns of the tile: a stage filled by two
  // terms instead of one piece per term)
  int64_t src2;
  int32_t elems2;
  int32_t pad;
};

struct DevTask {
  int32_t type;
  int32_t r0, r1;      // rows [r0,r1) of the block (Y) or slots (T)
  int32_t term0, nterm;  // Y: term range; T: term0 = the term instance
  int32_t eye0, neye;
  int32_t wait0, nwait;
  int32_t signal;      // counter to bump when done (-1: none)
  int32_t has_init;
  int32_t has_rhs;
  VecRef out;          // Y: output block start
  VecRef init;         // Y: partial sum to start from
  VecRef rhs;          // Y: + rhs_coef * rhs
  double rhs_coef;
  int32_t item0, nitem;    // per-column (Y_PLR) / per-slot (T_PLR) items
  int32_t piece0, npiece;  // operator ranges staged into smem
  int32_t run0, nrun;      // Y_PLR: runs of contiguous t values
  int32_t ncol;            // Y_PLR: flat columns of the task
  int32_t c0, c1;          // T_PLR: source columns [c0, c1) its Vt rows read
  int32_t tbase;           // T_PLR: SLOT_T index of the task's first Vt row
  int32_t q;               // queue index (set in the executor's metadata blob)
  int32_t srun0, nsrun;    // Y_PLR: runs of dense-leaf source columns
  int32_t ndense2;         // Y_PLR: second-source values those runs stage
};

// Per-task metadata item, 8 bytes, precomputed on the host.
//  Y_PLR column: U data at its piece + poff, tile rows [lo, hi).
//  T_PLR Vt row: data at its piece + poff, n columns, source at staged-slice
//                offset lo; result to SLOT_T[tbase + hi].
struct DevItem {
  uint16_t poff;
  uint16_t lo;
  uint16_t hi;
  uint16_t n;
};
static_assert(sizeof(DevItem) == 8, "DevItem is 8 bytes");
static_assert(sizeof(DevTask) % 16 == 0, "DevTask is copied in 16-byte words");

// Y_PLR: the t values of flat columns [f, f + n) are SLOT_T[t .. t + n)
struct DevRun {
  int32_t t;
  int16_t f;
  int16_t n;
};

// Y_PLR, dense leaf (a leaf whose U.Vt is stored as its product): the flat
// columns [f, f + n) take scale * (x_a + x_b) of source columns [col, col + n)
// of term `term`; x_b lands at staged offset nitem + b_off first
struct DevSrcRun {
  int32_t col;
  int16_t f;
  int16_t n;
  int16_t term;
  int16_t b_off;
  int32_t pad;
};

// PLR storage on the device.  For each leaf the factors are stored as
// rank "slots": slot c holds U[:, c] (rows contiguous, i.e. U column-major)
// and Vt[c, :] (cols contiguous).
struct DevLeaf {
  int64_t u_off;   // complex offset of U column 0 (column-major rows x rank)
  int64_t v_off;   // complex offset of Vt row 0 (row-major rank x cols)
  int32_t row_off, col_off, rows, cols, rank, slot0;  // slot0 within kernel
};

struct DevSlot {     // one Vt row, for the t-phase
  int64_t v_off;     // complex offset of this Vt row
  int32_t col_off, cols;
};

// T_PLR: a Vt row of n columns is reduced by 32, 16 or 8 consumer lanes
// (class 0, 1, 2), about 4-8 columns per lane
#ifdef __CUDACC__
__host__ __device__
#endif
inline int t_lane_class(int n) { return n > 160 ? 0 : n > 64 ? 1 : 2; }

constexpr int PLR_TILE = 16;           // rows of a Y_PLR task
constexpr int ROW_CHUNK = 64;          // output rows published per producer group
// per-task staging limits of the executor's task slots (defaults; the handle
// sizes its slots from the operator, see pt_create)
constexpr int MAX_T_SLOTS = 256;  // Vt rows (items) of one T_PLR task
constexpr int MAX_TCOLS = 256;    // source columns a T_PLR task stages (or its widest Vt row)

struct DevKernelPLR {
  int32_t leaf0, nleaf;      // into the leaf table
  int32_t slot0, nslot;      // into the slot table (nslot = sum of ranks)
  int32_t tile0;             // leaves meeting row tile t: tile_ent[tile_ptr[tile0+t] ..
  int32_t pad;               //                                  tile_ptr[tile0+t+1])
};

// One leaf as seen from one PLR_TILE-row tile.  U is stored tile-major: for
// each tile, each leaf meeting it, each rank column, the tile's rows of that
// column (hi - lo values).  Tile row r (lo <= r < hi) of column c is at
// u0 + c*stride + (r - lo), stride = hi - lo, u0 an absolute factor offset.
// A dense leaf (t0 = -1: one whose factors hold more bytes than U.Vt itself,
// e.g. the full-rank near-diagonal leaves) stores the tile's rows of U.Vt
// instead, its "rank" columns being the leaf's columns (rank = cols).
struct DevTileEntry {
  int64_t u0;
  int32_t t0;      // first slot of the leaf (kernel-relative; -1: dense leaf)
  int32_t stride;  // leaf rows (U is column-major)
  int32_t rank;
  int32_t pre;     // dense leaf (t0 < 0): its first column in the block
  int16_t lo, hi;
  int32_t pad;
};

}  // namespace pt
