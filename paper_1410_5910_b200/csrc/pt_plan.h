// Host-side operator description and program (task DAG) builder.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "pt_types.h"

namespace pt {

struct HostEntry {
  int64_t row, col, kernel;
  double s_re, s_im, e_re, e_im;
};

// The validated operator: entry table of the polarized system, the sweep
// permutation and the per-kernel storage description.
struct Operator {
  int64_t m = 0;   // block size
  int64_t nb = 0;  // block rows = block cols = 2*nt
  int64_t nt = 0;
  int fmt = 0;     // PT_KERNEL_DENSE / PT_KERNEL_PLR
  int nk = 0;
  std::vector<HostEntry> entries;  // sorted by (row, col)
  std::vector<int64_t> perm, inv;
  std::vector<int64_t> kernel_bytes;  // algorithmic bytes per kernel
  // PLR device-format tables (built by build_plr_tables)
  std::vector<DevLeaf> leaves;
  std::vector<DevSlot> slots;
  std::vector<DevKernelPLR> kplr;
  std::vector<int32_t> tile_ptr;
  std::vector<DevTileEntry> tile_ent;
  std::vector<int64_t> tile_chunk;  // per (kernel, tile): offset of its U chunk
  std::vector<int32_t> nslot;  // per kernel: sum of ranks
};

struct Program {
  std::vector<DevTask> tasks;
  std::vector<DevTerm> terms;
  std::vector<DevEye> eyes;
  std::vector<DevWait> waits;
  std::vector<DevTileEntry> ents;  // Y_PLR task entries (t0 absolute, pre = prefix)
  std::vector<DevPiece> pieces;    // staged operator ranges of every task
  std::vector<DevItem> items;      // per-task metadata items
  std::vector<DevRun> runs;        // Y_PLR t-value runs
  std::vector<DevSrcRun> sruns;    // Y_PLR dense-leaf source runs
  std::vector<uint8_t> chain;      // per task (queue order): on a sweep's dependency chain
  int n_counters = 0;
  int64_t t_elems = 0;      // size of SLOT_T needed
  int64_t term_bytes = 0;   // kernel bytes actually streamed by the terms
  int64_t algo_bytes = 0;   // distinct kernels per apply/sweep
  int64_t slot_elems[N_SLOTS] = {0};  // minimum size of each slot vector
  std::string overflow;     // non-empty: why a task exceeds the executor's staging (not runnable)
  std::string describe() const;
};

// Validation mirrors the reference's errors (ValueError -> false + msg).
bool validate_operator(Operator& op, std::string& err);
// "" or the ValueError message a sweep over this operator raises
std::string sweep_diagonal_error(const Operator& op);

// Program kinds.
struct PlanParams {
  int ctas = 444;                // executor CTAs (queue-order simulation)
  int64_t half_elems = 1024;     // complex capacity of one operator piece stage
  double task_us = 2.0;          // fixed cost per task in the simulation
  double cta_gbs = 25.0;         // streaming rate of one CTA in the simulation
  int dense_rows_per_task = 16;  // Y_DENSE rows per task
  int plr_rows_per_task = PLR_TILE;  // Y_PLR rows per task (lane per row)
  int plr_slots_per_task = 64;   // T_PLR slots per task (warp per slot)
  int t_pieces = 2;              // ring-stage pieces per T_PLR task
  int t_pieces_chain = 1;        // ... in the sweeps' dependency chain
  int row_chunk = ROW_CHUNK;     // output rows published per producer group
  int64_t item_cap = 1 << 20;    // metadata items a task slot holds
  bool piece_pairs = false;      // a Y_PLR ring stage may hold the columns of two terms (two ranges)
  int max_block_terms = 0;       // A-apply: kernel terms per output task (0: all; else a block row is
                                 // emitted as partial sums of at most this many terms: smaller task slots)
  bool force_dense = false;      // plan row-major dense tasks (Y_DENSE) whatever the operator's storage
                                 // (the batched executor streams the row-major dense pool)
  int64_t tcols_cap = MAX_TCOLS; // source columns a T_PLR task stages
};

Program build_apply_A(const Operator& op, const PlanParams& pp);
// n_it sweeps from zero on rhs = SLOT_IN (preconditioner_apply).
Program build_apply_M(const Operator& op, int n_it, const PlanParams& pp);
// one sweep: rhs = SLOT_IN, u_in = SLOT_AUX (gs_sweep)
Program build_gs_sweep(const Operator& op, const PlanParams& pp);
// w = M^-1 (A x): x = SLOT_IN, result in SLOT_OUT (one GMRES iteration)
Program build_A_then_M(const Operator& op, int n_it, const PlanParams& pp);

}  // namespace pt
