// Host plan builder: turns the polarized entry table into task DAGs.
//
// Reference semantics restated here (file:line in pkg/src/helmsweep/):
//  * A-apply  y_i = sum_j scale_ij K_ij x_j + eye_ij x_j
//    (BlockInterfaceMatrix.matvec / BlockEntry.apply, trace_system.py:159-226)
//  * split_DR (trace_system.py:499-524): row i goes to position inv[i] of the
//    sweep permutation; down rows x down cols -> D_down, x up cols -> R_up,
//    up rows x down cols -> R_down, x up cols -> D_up.
//  * gs_sweep (solver.py:203-220) + solve_block_triangular
//    (trace_system.py:527-548): x_p = sum_{j != p} D_pj x_j + (R u)_p - rhs_p,
//    ascending for the down half, descending for the up half; a diagonal
//    that is not exactly -I raises; entries on the not-yet-solved side
//    multiply the zero-initialised x and contribute nothing.
//
// B200-specific restructuring (results equal up to rounding):
//  * kernel terms of one block row that share a kernel and a scale are
//    merged, K (x_a + x_b): in the A-apply this is K (x_down + x_up); in a
//    sweep it is the D kernel applied to (x_new + u_old) of the R entry at
//    the same block position, so every distinct kernel is streamed once per
//    apply;
//  * R-only terms of a sweep go to a pre-phase partial sum that does not
//    wait for the sequential chain; the chain task starts from it;
//  * sweep 1 starts from u = 0, so its R terms are skipped (bitwise exact).
#include "pt_plan.h"

#include <algorithm>
#include <climits>
#include <cmath>
#include <map>
#include <queue>
#include <set>
#include <sstream>

namespace pt {

namespace {

struct TermSpec {
  int64_t kernel;
  double s_re, s_im;
  std::vector<VecRef> src;
};
struct EyeSpec {
  double re, im;
  VecRef src;
};

VecRef ref(int32_t slot, int64_t off) {
  VecRef r;
  r.slot = slot;
  r.pad = 0;
  r.off = off;
  return r;
}

class Builder {
 public:
  Builder(const Operator& op, const PlanParams& pp) : op_(op), pp_(pp) {}
  // pieces per T_PLR task for the blocks emitted next (0: pp.t_pieces)
  int t_pieces_now = 0;
  // the blocks emitted next are on a sweep's dependency chain (queue priority)
  bool chain_now = false;
  const PlanParams& params() const { return pp_; }
  // operator elements per T_PLR piece: one ring stage
  int64_t t_piece_cap() const { return pp_.half_elems; }

  int emit_block(VecRef out, const std::vector<TermSpec>& terms,
                 const std::vector<EyeSpec>& eyes, bool has_init, VecRef init,
                 bool has_rhs, VecRef rhs, double rhs_coef) {
    // waits every output task of the block has (t-vectors, dense sources);
    // the row-local inputs (eyes, init, rhs) are added per task
    std::vector<int> waits;
    // producers of init as they are now: a block that accumulates in place
    // (init == out) replaces them below
    std::vector<RowGroup> init_prod;
    if (has_init) {
      auto it = producer_.find(std::make_pair(init.slot, init.off));
      if (it != producer_.end()) init_prod = it->second;
    }
    const int32_t term0 = (int32_t)prog_.terms.size();
    const bool plr = op_.fmt == 1 && !pp_.force_dense && !terms.empty();
    double ybytes = 0.0;
    for (const TermSpec& t : terms) {
      DevTerm dt{};
      dt.kernel = (int32_t)t.kernel;
      dt.nsrc = (int32_t)t.src.size();
      dt.scale_re = t.s_re;
      dt.scale_im = t.s_im;
      for (size_t s = 0; s < t.src.size(); ++s) dt.src[s] = t.src[s];
      dt.t_base = -1;
      sweep_kernels_.insert(t.kernel);
      prog_.term_bytes += op_.kernel_bytes[t.kernel];
      if (plr) {
        const int32_t ns = op_.nslot[t.kernel];
        dt.t_base = alloc_t(ns);
        // T tasks: t = Vt (sum of sources); each waits only for the source
        // rows its slice [c0, c1) reads
        const int g = new_group();
        const int32_t term_idx = (int32_t)prog_.terms.size();
        const DevKernelPLR& kp = op_.kplr[t.kernel];
        for (int32_t s0 = 0; s0 < ns;) {
          // slots whose Vt rows fill at most one smem buffer half
          // up to T_PIECES pieces, each a run of slots filling one buffer half
          DevTask tk{};
          tk.type = TASK_T_PLR;
          tk.r0 = s0;
          tk.term0 = term_idx;
          tk.nterm = 1;
          tk.piece0 = (int32_t)prog_.pieces.size();
          int32_t s1 = s0;
          int64_t total = 0;
          const int32_t cap = (int32_t)std::min<int64_t>(pp_.plr_slots_per_task, pp_.item_cap);
          int32_t span0 = INT32_MAX, span1 = INT32_MIN;
          bool span_full = false;
          const int tp = t_pieces_now > 0 ? t_pieces_now : pp_.t_pieces;
          for (int np = 0; np < tp && s1 < ns && s1 - s0 < cap && !span_full; ++np) {
            DevPiece pc{};
            pc.src = op_.slots[kp.slot0 + s1].v_off;
            pc.f0 = s1 - s0;
            int64_t elems = 0;
            while (s1 < ns && s1 - s0 < cap) {
              const DevSlot& sl = op_.slots[kp.slot0 + s1];
              const int64_t c = sl.cols;
              if (s1 - s0 > pc.f0 && elems + c > t_piece_cap()) break;
              // the staged source slice [c0, c1) of the task stays within tcols_cap
              const int32_t lo = std::min(span0, sl.col_off);
              const int32_t hi = std::max(span1, sl.col_off + sl.cols);
              if (s1 > s0 && hi - lo > pp_.tcols_cap) {
                span_full = true;
                break;
              }
              span0 = lo;
              span1 = hi;
              elems += c;
              ++s1;
            }
            if (s1 - s0 == pc.f0) break;  // nothing fits next to the staged slice
            if (elems > pp_.half_elems) flag("a Vt row exceeds an operator stage");
            pc.elems = (int32_t)elems;
            pc.f1 = s1 - s0;
            // consumer lanes per Vt row: 32, 16 or 8 by the row's own length
            // (~4-8 columns per lane); the piece's items are ordered by lane
            // class below, counts packed in e0 (t_lane_classes)
            int32_t ncls[3] = {0, 0, 0};
            for (int32_t q = s0 + pc.f0; q < s1; ++q) ncls[t_lane_class(op_.slots[kp.slot0 + q].cols)]++;
            pc.e0 = ncls[0] | (ncls[1] << 10) | (ncls[2] << 20);
            prog_.pieces.push_back(pc);
            total += elems;
          }
          tk.r1 = s1;
          tk.npiece = (int32_t)prog_.pieces.size() - tk.piece0;
          tk.c0 = (int32_t)op_.m;
          tk.c1 = 0;
          for (int32_t q = s0; q < s1; ++q) {
            const DevSlot& sl = op_.slots[kp.slot0 + q];
            tk.c0 = std::min(tk.c0, sl.col_off);
            tk.c1 = std::max(tk.c1, sl.col_off + sl.cols);
          }
          // one item per slot: Vt row offset within its piece, source offset
          // within the staged slice, destination in SLOT_T
          tk.item0 = (int32_t)prog_.items.size();
          tk.tbase = (int32_t)(dt.t_base + s0);
          for (int32_t p = 0; p < tk.npiece; ++p) {
            const DevPiece& pc = prog_.pieces[tk.piece0 + p];
            for (int cls = 0; cls < 3; ++cls) {  // 32-lane rows, then 16, then 8
              for (int32_t q = pc.f0; q < pc.f1; ++q) {
                const DevSlot& sl = op_.slots[kp.slot0 + s0 + q];
                if (t_lane_class(sl.cols) != cls) continue;
                DevItem it{};
                it.poff = (uint16_t)(sl.v_off - pc.src);
                it.lo = (uint16_t)(sl.col_off - tk.c0);
                it.hi = (uint16_t)q;  // the row's slot within the task
                it.n = (uint16_t)sl.cols;
                prog_.items.push_back(it);
              }
            }
          }
          tk.nitem = (int32_t)prog_.items.size() - tk.item0;
          if (tk.nitem > pp_.item_cap) flag("a T task has more slots than a task slot holds");
          if (tk.c1 - tk.c0 > pp_.tcols_cap) flag("a Vt row is wider than a task slot stages");
          std::vector<int> twaits;
          for (const VecRef& sv : t.src) add_wait_rows(twaits, sv, tk.c0, tk.c1);
          push_task(tk, twaits, g, 16.0 * (double)total);
          s0 = s1;
        }
        register_producer(ref(SLOT_T, dt.t_base), g);
        add_wait(waits, ref(SLOT_T, dt.t_base));
        ybytes += 0.5 * (double)op_.kernel_bytes[t.kernel];
      } else {
        for (const VecRef& s : t.src) add_wait(waits, s);
        ybytes += (double)op_.kernel_bytes[t.kernel];
      }
      prog_.terms.push_back(dt);
    }
    const int32_t eye0 = (int32_t)prog_.eyes.size();
    for (const EyeSpec& e : eyes) {
      DevEye de{};
      de.re = e.re;
      de.im = e.im;
      de.src = e.src;
      prog_.eyes.push_back(de);
    }
    // output rows are published in chunks of ROW_CHUNK rows (one producer
    // group each), so consumers of a row range start before the block ends
    const int64_t m = op_.m;
    const int rpt = plr ? pp_.plr_rows_per_task : pp_.dense_rows_per_task;
    const int64_t chunk_rows = std::max<int64_t>(pp_.row_chunk / rpt, 1) * rpt;
    int g = -1;
    for (int64_t r0 = 0; r0 < m; r0 += rpt) {
      std::vector<int> dense_waits;  // source rows the task's dense leaves read
      if (r0 % chunk_rows == 0) {
        g = new_group();
        register_producer_rows(out, r0, std::min<int64_t>(m, r0 + chunk_rows), g);
      }
      DevTask tk{};
      tk.piece0 = (int32_t)prog_.pieces.size();
      if (plr) {  // one item per flat (leaf, rank column) of all terms, pieces of whole columns
        tk.item0 = (int32_t)prog_.items.size();
        tk.run0 = (int32_t)prog_.runs.size();
        tk.srun0 = (int32_t)prog_.sruns.size();
        int32_t f = 0, dense2 = 0;
        // A piece is one ring stage: a contiguous range of the tile's columns
        // of one term, and, where it fits, a second range (the next term's
        // columns) right behind it (pp_.piece_pairs).
        DevPiece pc{};
        bool open = false, in_second = false;
        for (size_t it = 0; it < terms.size(); ++it) {
          const DevTerm& dt = prog_.terms[term0 + it];
          const int32_t k0 = op_.kplr[dt.kernel].tile0 + (int32_t)(r0 / PLR_TILE);
          bool first_of_term = true;
          int64_t term_elems = 0;  // the term's columns of this tile
          for (int32_t e = op_.tile_ptr[k0]; e < op_.tile_ptr[k0 + 1]; ++e)
            term_elems += (int64_t)op_.tile_ent[e].rank * op_.tile_ent[e].stride;
          for (int32_t e = op_.tile_ptr[k0]; e < op_.tile_ptr[k0 + 1]; ++e) {
            const DevTileEntry& te = op_.tile_ent[e];
            if (te.rank > 0 && te.t0 >= 0) {  // t values from the term's T tasks
              DevRun run{};
              run.t = (int32_t)(dt.t_base + te.t0);
              run.f = (int16_t)f;
              run.n = (int16_t)te.rank;
              prog_.runs.push_back(run);
            } else if (te.rank > 0) {  // dense leaf: scaled source columns
              DevSrcRun sr{};
              sr.col = te.pre;
              sr.f = (int16_t)f;
              sr.n = (int16_t)te.rank;
              sr.term = (int16_t)it;
              sr.b_off = (int16_t)dense2;
              if (dt.nsrc > 1) dense2 += te.rank;
              prog_.sruns.push_back(sr);
              for (int sidx = 0; sidx < dt.nsrc; ++sidx)
                add_wait_rows(dense_waits, dt.src[sidx], te.pre, te.pre + te.rank);
            }
            for (int32_t c = 0; c < te.rank; ++c, ++f) {
              const int64_t addr = te.u0 + (int64_t)c * te.stride;
              // the open piece takes the column if it fits and continues one
              // of its ranges -- or starts its second range (a new term)
              const bool fits = open && pc.elems + pc.elems2 + te.stride <= pp_.half_elems;
              const bool contiguous =
                  open && addr == (in_second ? pc.src2 + pc.elems2 : pc.src + pc.elems);
              // (a second range only for a term that fits whole: no fragments of large terms)
              const bool second = open && !contiguous && first_of_term && !in_second &&
                                  pp_.piece_pairs && pc.elems + term_elems <= pp_.half_elems;
              if (open && !(fits && (contiguous || second))) {
                prog_.pieces.push_back(pc);
                open = false;
              }
              if (!open) {
                pc = DevPiece{};
                pc.src = addr;
                pc.f0 = f;
                open = true;
                in_second = false;
              } else if (!contiguous) {
                pc.src2 = addr;
                in_second = true;
              }
              first_of_term = false;
              DevItem item{};
              item.poff = (uint16_t)(pc.elems + pc.elems2);
              item.lo = (uint16_t)te.lo;
              item.hi = (uint16_t)te.hi;
              item.n = 0;
              prog_.items.push_back(item);
              (in_second ? pc.elems2 : pc.elems) += te.stride;
              pc.f1 = f + 1;
            }
          }
        }
        if (open) prog_.pieces.push_back(pc);
        tk.nitem = (int32_t)prog_.items.size() - tk.item0;
        tk.nrun = (int32_t)prog_.runs.size() - tk.run0;
        tk.nsrun = (int32_t)prog_.sruns.size() - tk.srun0;
        tk.ndense2 = dense2;
        tk.ncol = f;
        if (tk.nitem > pp_.item_cap) flag("a PLR row tile has more rank columns than a task slot holds");
      } else {
        for (size_t it = 0; it < terms.size(); ++it) {
          DevPiece pc{};
          pc.src = ((int64_t)terms[it].kernel * m + r0) * m;
          pc.elems = (int32_t)((std::min<int64_t>(m, r0 + rpt) - r0) * m);
          pc.f0 = (int32_t)it;
          pc.f1 = (int32_t)it + 1;
          if (pc.elems > pp_.half_elems) flag("dense kernel rows exceed an operator stage");
          prog_.pieces.push_back(pc);
        }
      }
      tk.npiece = (int32_t)prog_.pieces.size() - tk.piece0;
      tk.c0 = 0;
      tk.c1 = (int32_t)m;
      tk.type = plr ? TASK_Y_PLR : TASK_Y_DENSE;
      tk.r0 = (int32_t)r0;
      tk.r1 = (int32_t)std::min<int64_t>(m, r0 + rpt);
      tk.term0 = term0;
      tk.nterm = (int32_t)terms.size();
      tk.eye0 = eye0;
      tk.neye = (int32_t)eyes.size();
      tk.out = out;
      tk.has_init = has_init ? 1 : 0;
      tk.init = init;
      tk.has_rhs = has_rhs ? 1 : 0;
      tk.rhs = rhs;
      tk.rhs_coef = rhs_coef;
      std::vector<int> tw = waits;
      for (int g2 : dense_waits)
        if (std::find(tw.begin(), tw.end(), g2) == tw.end()) tw.push_back(g2);
      for (const EyeSpec& e : eyes) add_wait_rows(tw, e.src, tk.r0, tk.r1);
      if (has_init)
        for (const RowGroup& rg : init_prod)
          if (rg.lo < tk.r1 && tk.r0 < rg.hi && std::find(tw.begin(), tw.end(), rg.g) == tw.end())
            tw.push_back(rg.g);
      if (has_rhs) add_wait_rows(tw, rhs, tk.r0, tk.r1);
      push_task(tk, tw, g, ybytes * double(tk.r1 - tk.r0) / double(m));
    }
    return g;
  }

  bool overflow() const { return !overflow_.empty(); }
  void flag(const char* why) {
    if (overflow_.empty()) overflow_ = why;
  }
  void begin_stage() { sweep_kernels_.clear(); }
  void end_stage() {
    for (int64_t k : sweep_kernels_) prog_.algo_bytes += op_.kernel_bytes[k];
    sweep_kernels_.clear();
  }

  void need_slot(int32_t slot, int64_t elems) {
    prog_.slot_elems[slot] = std::max(prog_.slot_elems[slot], elems);
  }

  Program finish() {
    const int n = (int)prog_.tasks.size();
    // modelled duration of each task on one CTA
    std::vector<double> dur(n);
    for (int t = 0; t < n; ++t) dur[t] = pp_.task_us + task_cost_[t] / (pp_.cta_gbs * 1e3);
    // bottom level = duration-weighted longest path to a sink (priority)
    std::vector<double> bl(n, 0.0), gcons(groups_.size(), 0.0);
    for (int t = n - 1; t >= 0; --t) {
      bl[t] = dur[t] + gcons[task_group_[t]];
      for (int g : task_waits_[t]) gcons[g] = std::max(gcons[g], bl[t]);
    }
    // List-scheduling simulation on pp_.ctas CTAs: a task is released when
    // all its producer groups have finished; a free CTA takes the released
    // task with the longest remaining path.  The queue order is the
    // simulated start order, so CTAs grabbing in queue order interleave
    // independent groups the way the schedule does (topological by
    // construction: a task starts after its producers finish).
    std::vector<int> unmet(n), gleft(groups_.size(), 0);
    std::vector<std::vector<int>> gcons_list(groups_.size());
    for (int t = 0; t < n; ++t) {
      gleft[task_group_[t]]++;
      unmet[t] = (int)task_waits_[t].size();
      for (int g : task_waits_[t]) gcons_list[g].push_back(t);
    }
    typedef std::pair<double, int> PI;
    std::priority_queue<PI> ready;  // (bottom level, -index)
    std::priority_queue<PI, std::vector<PI>, std::greater<PI>> running;  // (finish, task)
    for (size_t g = 0; g < groups_.size(); ++g)  // empty groups are complete at once
      if (gleft[g] == 0)
        for (int c : gcons_list[g]) --unmet[c];
    // (a queue-priority bonus for the sweeps' chain tasks measured slower)
    auto prio = [&](int t) { return bl[t]; };
    for (int t = 0; t < n; ++t)
      if (unmet[t] == 0) ready.push(PI(prio(t), -t));
    std::vector<int> order;
    order.reserve(n);
    int busy = 0;
    double now = 0.0;
    while ((int)order.size() < n) {
      while (busy < pp_.ctas && !ready.empty()) {
        const int t = -ready.top().second;
        ready.pop();
        order.push_back(t);
        running.push(PI(now + dur[t], t));
        ++busy;
      }
      if (running.empty()) {  // cannot happen for a DAG; keep every task regardless
        for (int t = 0; t < n; ++t)
          if (std::find(order.begin(), order.end(), t) == order.end()) order.push_back(t);
        break;
      }
      const PI ev = running.top();
      running.pop();
      --busy;
      now = ev.first;
      const int g = task_group_[ev.second];
      if (--gleft[g] == 0)
        for (int c : gcons_list[g])
          if (--unmet[c] == 0) ready.push(PI(prio(c), -c));
    }
    Program out;
    out.overflow = overflow_;
    out.terms = prog_.terms;
    out.eyes = prog_.eyes;
    out.ents = prog_.ents;
    out.pieces = prog_.pieces;
    out.items = prog_.items;
    out.runs = prog_.runs;
    out.sruns = prog_.sruns;
    out.t_elems = prog_.t_elems;
    out.term_bytes = prog_.term_bytes;
    out.algo_bytes = prog_.algo_bytes;
    for (int s = 0; s < N_SLOTS; ++s) out.slot_elems[s] = prog_.slot_elems[s];
    out.slot_elems[SLOT_T] = std::max<int64_t>(out.slot_elems[SLOT_T], prog_.t_elems);
    out.n_counters = (int)groups_.size();
    for (int idx : order) {
      DevTask tk = prog_.tasks[idx];
      tk.wait0 = (int32_t)out.waits.size();
      tk.nwait = (int32_t)task_waits_[idx].size();
      for (int g : task_waits_[idx]) {
        DevWait w;
        w.ctr = groups_[g].ctr;
        w.val = groups_[g].count;
        out.waits.push_back(w);
      }
      out.tasks.push_back(tk);
      out.chain.push_back(task_chain_[idx] ? 1 : 0);
    }
    return out;
  }

 private:
  struct Group {
    int ctr;
    int count;
  };

  int new_group() {
    Group g;
    g.ctr = (int)groups_.size();
    g.count = 0;
    groups_.push_back(g);
    return g.ctr;
  }

  // producer groups of a vector block, by row range (a later producer of the
  // same block replaces the earlier ones)
  struct RowGroup {
    int64_t lo, hi;
    int g;
  };
  void register_producer(VecRef block, int g) {
    producer_[std::make_pair(block.slot, block.off)] = {RowGroup{0, INT64_MAX, g}};
  }
  void register_producer_rows(VecRef block, int64_t lo, int64_t hi, int g) {
    auto& v = producer_[std::make_pair(block.slot, block.off)];
    if (lo == 0) v.clear();
    v.push_back(RowGroup{lo, hi, g});
  }

  void add_wait(std::vector<int>& waits, VecRef r) { add_wait_rows(waits, r, 0, INT64_MAX); }
  // wait for the producers of rows [lo, hi) of block r
  void add_wait_rows(std::vector<int>& waits, VecRef r, int64_t lo, int64_t hi) {
    auto it = producer_.find(std::make_pair(r.slot, r.off));
    if (it == producer_.end()) return;
    for (const RowGroup& rg : it->second)
      if (rg.lo < hi && lo < rg.hi && std::find(waits.begin(), waits.end(), rg.g) == waits.end())
        waits.push_back(rg.g);
  }

  int64_t alloc_t(int64_t n) {
    const int64_t base = prog_.t_elems;
    prog_.t_elems += (n + 7) / 8 * 8;
    return base;
  }

  void push_task(DevTask tk, const std::vector<int>& waits, int g, double cost) {
    tk.signal = groups_[g].ctr;
    groups_[g].count += 1;
    prog_.tasks.push_back(tk);
    task_waits_.push_back(waits);
    task_group_.push_back(g);
    task_cost_.push_back(cost);
    task_chain_.push_back(chain_now);
  }

  const Operator& op_;
  PlanParams pp_;
  Program prog_;
  std::map<std::pair<int32_t, int64_t>, std::vector<RowGroup>> producer_;
  std::vector<Group> groups_;
  std::vector<std::vector<int>> task_waits_;
  std::vector<int> task_group_;
  std::vector<double> task_cost_;
  std::vector<bool> task_chain_;
  std::set<int64_t> sweep_kernels_;
  std::string overflow_;  // why the program cannot run (empty: it can)
};

bool same_scale(const TermSpec& t, const HostEntry& e) {
  return t.kernel == e.kernel && t.s_re == e.s_re && t.s_im == e.s_im;
}

// A-apply: one output block per natural block row.
void emit_A(Builder& b, const Operator& op, int32_t in_slot, int32_t out_slot) {
  const int64_t m = op.m;
  b.begin_stage();
  b.need_slot(out_slot, op.nb * m);
  size_t k = 0;
  for (int64_t i = 0; i < op.nb; ++i) {
    std::vector<TermSpec> terms;
    std::vector<EyeSpec> eyes;
    for (; k < op.entries.size() && op.entries[k].row == i; ++k) {
      const HostEntry& e = op.entries[k];
      const VecRef src = ref(in_slot, e.col * m);
      if (e.kernel >= 0) {
        bool merged = false;
        for (TermSpec& t : terms) {
          if (same_scale(t, e) && t.src.size() < 2) {
            t.src.push_back(src);
            merged = true;
            break;
          }
        }
        if (!merged) terms.push_back(TermSpec{e.kernel, e.s_re, e.s_im, {src}});
      }
      if (e.e_re != 0.0 || e.e_im != 0.0) eyes.push_back(EyeSpec{e.e_re, e.e_im, src});
    }
    const int cap = b.params().max_block_terms;
    if (op.fmt == 1 && !b.params().force_dense && cap > 0 && (int)terms.size() > cap) {
      // partial sums of at most `cap` terms, accumulated in place; heavy and
      // light kernels paired so the partial tasks stage about the same
      std::sort(terms.begin(), terms.end(), [&](const TermSpec& x, const TermSpec& y) {
        return op.kernel_bytes[x.kernel] > op.kernel_bytes[y.kernel];
      });
      const int nparts = ((int)terms.size() + cap - 1) / cap;
      std::vector<std::vector<TermSpec>> parts(nparts);
      for (size_t t = 0; t < terms.size(); ++t) {
        const size_t round = t / nparts, pos = t % nparts;
        parts[round % 2 == 0 ? pos : nparts - 1 - pos].push_back(terms[t]);
      }
      const VecRef out = ref(out_slot, i * m);
      for (int p = 0; p < nparts; ++p)
        b.emit_block(out, parts[p], p == nparts - 1 ? eyes : std::vector<EyeSpec>(), p > 0, out, false,
                     VecRef{}, 0.0);
    } else {
      b.emit_block(ref(out_slot, i * m), terms, eyes, false, VecRef{}, false, VecRef{}, 0.0);
    }
  }
  b.end_stage();
}

struct HalfEntry {
  const HostEntry* e;
  int64_t jj;  // block column within its half
  bool is_d;
};

// One Gauss-Seidel sweep u_new = D^-1 (P rhs - R u_old).
void emit_sweep(Builder& b, const Operator& op, VecRef rhs, bool has_uold, VecRef uold,
                VecRef unew, VecRef pre) {
  const int64_t m = op.m, nt = op.nt;
  b.begin_stage();
  // small T tasks for the whole sweep: its pre-phase tasks share CTAs with
  // the chain and must not hold a CTA's consumers long
  b.t_pieces_now = b.params().t_pieces_chain;
  b.need_slot(unew.slot, unew.off + op.nb * m);
  b.need_slot(pre.slot, pre.off + op.nb * m);
  // rows[h][p]: entries of half-row p
  std::vector<std::vector<HalfEntry>> rows[2];
  rows[0].resize(nt);
  rows[1].resize(nt);
  for (const HostEntry& e : op.entries) {
    const int64_t pos = op.inv[e.row];
    const int h = pos >= nt ? 1 : 0;
    const int64_t p = pos - h * nt;
    const int colhalf = e.col >= nt ? 1 : 0;
    rows[h][p].push_back(HalfEntry{&e, e.col - colhalf * nt, colhalf == h});
  }
  auto unew_ref = [&](int h, int64_t j) { return ref(unew.slot, unew.off + (h * nt + j) * m); };
  auto uold_ref = [&](int h, int64_t j) {
    return ref(uold.slot, uold.off + ((1 - h) * nt + j) * m);
  };
  // levels
  std::vector<int> level[2];
  for (int h = 0; h < 2; ++h) {
    level[h].assign(nt, 0);
    for (int64_t q = 0; q < nt; ++q) {
      const int64_t p = h == 0 ? q : nt - 1 - q;
      int lv = 0;
      for (const HalfEntry& he : rows[h][p]) {
        if (!he.is_d) continue;
        const bool chain = h == 0 ? he.jj < p : he.jj > p;
        if (chain) lv = std::max(lv, level[h][he.jj] + 1);
      }
      level[h][p] = lv;
    }
  }
  int max_level = 0;
  for (int h = 0; h < 2; ++h)
    for (int v : level[h]) max_level = std::max(max_level, v);

  struct RowPlan {
    std::vector<TermSpec> chain_terms, r_terms;
    std::vector<EyeSpec> chain_eyes, r_eyes;
  };
  std::vector<RowPlan> plans[2];
  for (int h = 0; h < 2; ++h) {
    plans[h].resize(nt);
    for (int64_t p = 0; p < nt; ++p) {
      RowPlan& rp = plans[h][p];
      std::vector<TermSpec> rk;
      for (const HalfEntry& he : rows[h][p]) {
        const HostEntry& e = *he.e;
        if (he.is_d) {
          if (he.jj == p) continue;  // diagonal: validated -I (see validate)
          const bool chain = h == 0 ? he.jj < p : he.jj > p;
          if (!chain) continue;  // multiplies the zero-initialised x
          const VecRef src = unew_ref(h, he.jj);
          if (e.kernel >= 0) rp.chain_terms.push_back(TermSpec{e.kernel, e.s_re, e.s_im, {src}});
          if (e.e_re != 0.0 || e.e_im != 0.0) rp.chain_eyes.push_back(EyeSpec{e.e_re, e.e_im, src});
        } else if (has_uold) {
          const VecRef src = uold_ref(h, he.jj);
          if (e.kernel >= 0) rk.push_back(TermSpec{e.kernel, e.s_re, e.s_im, {src}});
          if (e.e_re != 0.0 || e.e_im != 0.0) rp.r_eyes.push_back(EyeSpec{e.e_re, e.e_im, src});
        }
      }
      // merge R kernel terms into chain terms with the same kernel and scale
      for (TermSpec& r : rk) {
        bool merged = false;
        for (TermSpec& c : rp.chain_terms) {
          if (c.kernel == r.kernel && c.s_re == r.s_re && c.s_im == r.s_im && c.src.size() == 1) {
            c.src.push_back(r.src[0]);
            merged = true;
            break;
          }
        }
        if (!merged) rp.r_terms.push_back(r);
      }
    }
  }
  // pre-phase: R-only terms - rhs, for rows that also have chain work
  std::vector<bool> has_pre[2];
  for (int h = 0; h < 2; ++h) {
    has_pre[h].assign(nt, false);
    for (int64_t p = 0; p < nt; ++p) {
      RowPlan& rp = plans[h][p];
      const bool chain = !rp.chain_terms.empty() || !rp.chain_eyes.empty();
      const bool ronly = !rp.r_terms.empty() || !rp.r_eyes.empty();
      if (chain && ronly) {
        has_pre[h][p] = true;
        const VecRef dst = ref(pre.slot, pre.off + (h * nt + p) * m);
        b.emit_block(dst, rp.r_terms, rp.r_eyes, false, VecRef{}, true,
                     ref(rhs.slot, rhs.off + op.perm[h * nt + p] * m), -1.0);
      }
    }
  }
  // chain, level by level, both halves interleaved (small T tasks: a level's
  // t-phase spreads over all CTAs; its latency is on the critical path)
  b.chain_now = true;
  for (int lv = 0; lv <= max_level; ++lv) {
    for (int h = 0; h < 2; ++h) {
      for (int64_t q = 0; q < nt; ++q) {
        const int64_t p = h == 0 ? q : nt - 1 - q;
        if (level[h][p] != lv) continue;
        RowPlan& rp = plans[h][p];
        const VecRef rhs_p = ref(rhs.slot, rhs.off + op.perm[h * nt + p] * m);
        if (has_pre[h][p]) {
          b.emit_block(unew_ref(h, p), rp.chain_terms, rp.chain_eyes, true,
                       ref(pre.slot, pre.off + (h * nt + p) * m), false, VecRef{}, 0.0);
        } else {
          std::vector<TermSpec> terms = rp.chain_terms;
          terms.insert(terms.end(), rp.r_terms.begin(), rp.r_terms.end());
          std::vector<EyeSpec> eyes = rp.chain_eyes;
          eyes.insert(eyes.end(), rp.r_eyes.begin(), rp.r_eyes.end());
          b.emit_block(unew_ref(h, p), terms, eyes, false, VecRef{}, true, rhs_p, -1.0);
        }
      }
    }
  }
  b.t_pieces_now = 0;
  b.chain_now = false;
  b.end_stage();
}

void emit_M(Builder& b, const Operator& op, int n_it, VecRef rhs) {
  const int64_t N = op.nb * op.m;
  bool has_old = false;
  VecRef uold{};
  for (int k = 0; k < n_it; ++k) {
    const VecRef out = (k == n_it - 1) ? ref(SLOT_OUT, 0) : ref(SLOT_U1, (int64_t)k * N);
    emit_sweep(b, op, rhs, has_old, uold, out, ref(SLOT_PRE, (int64_t)k * N));
    uold = out;
    has_old = true;
  }
}

}  // namespace

bool validate_operator(Operator& op, std::string& err) {
  std::ostringstream os;
  if (op.m <= 0) {
    err = "block size m must be positive";
    return false;
  }
  if (op.nb <= 0 || op.nb % 2) {
    err = "polarized matrix must be square with an even block count";
    return false;
  }
  op.nt = op.nb / 2;
  if ((int64_t)op.perm.size() != op.nb) {
    err = "sweep permutation has the wrong length";
    return false;
  }
  op.inv.assign(op.nb, -1);
  for (int64_t p = 0; p < op.nb; ++p) {
    const int64_t v = op.perm[p];
    if (v < 0 || v >= op.nb || op.inv[v] != -1) {
      err = "sweep permutation is not a permutation of the block rows";
      return false;
    }
    op.inv[v] = p;
  }
  std::sort(op.entries.begin(), op.entries.end(), [](const HostEntry& a, const HostEntry& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  for (size_t i = 0; i < op.entries.size(); ++i) {
    const HostEntry& e = op.entries[i];
    if (e.row < 0 || e.row >= op.nb || e.col < 0 || e.col >= op.nb) {
      os << "block (" << e.row << "," << e.col << ") outside " << op.nb << "x" << op.nb;
      err = os.str();
      return false;
    }
    if (i && op.entries[i - 1].row == e.row && op.entries[i - 1].col == e.col) {
      os << "block (" << e.row << "," << e.col << ") assigned twice";
      err = os.str();
      return false;
    }
    if (e.kernel < -1 || e.kernel >= op.nk) {
      os << "block (" << e.row << "," << e.col << ") references kernel " << e.kernel;
      err = os.str();
      return false;
    }
  }
  return true;
}

// A diagonal block of D that is not exactly -I makes the sweep raise
// (trace_system.py:542-544); returns the message or "".
std::string sweep_diagonal_error(const Operator& op) {
  for (const HostEntry& e : op.entries) {
    const int64_t pos = op.inv[e.row];
    const int h = pos >= op.nt ? 1 : 0;
    const int colhalf = e.col >= op.nt ? 1 : 0;
    if (colhalf != h) continue;
    const int64_t p = pos - h * op.nt, jj = e.col - colhalf * op.nt;
    if (jj == p && !(e.kernel < 0 && e.e_re == -1.0 && e.e_im == 0.0)) {
      std::ostringstream os;
      os << "diagonal block " << p << " is not exactly -I";
      return os.str();
    }
  }
  return "";
}

Program build_apply_A(const Operator& op, const PlanParams& pp) {
  Builder b(op, pp);
  emit_A(b, op, SLOT_IN, SLOT_OUT);
  return b.finish();
}

Program build_apply_M(const Operator& op, int n_it, const PlanParams& pp) {
  Builder b(op, pp);
  emit_M(b, op, n_it, ref(SLOT_IN, 0));
  return b.finish();
}

Program build_gs_sweep(const Operator& op, const PlanParams& pp) {
  Builder b(op, pp);
  emit_sweep(b, op, ref(SLOT_IN, 0), true, ref(SLOT_AUX, 0), ref(SLOT_OUT, 0), ref(SLOT_PRE, 0));
  return b.finish();
}

Program build_A_then_M(const Operator& op, int n_it, const PlanParams& pp) {
  Builder b(op, pp);
  emit_A(b, op, SLOT_IN, SLOT_Y);
  emit_M(b, op, n_it, ref(SLOT_Y, 0));
  return b.finish();
}

std::string Program::describe() const {
  std::ostringstream os;
  int counts[3] = {0, 0, 0};
  for (const DevTask& t : tasks) counts[t.type]++;
  os << tasks.size() << " tasks (Ydense " << counts[0] << ", Yplr " << counts[1] << ", Tplr "
     << counts[2] << "), " << terms.size() << " terms, " << n_counters << " counters, algo "
     << algo_bytes << " B, streamed " << term_bytes << " B";
  return os.str();
}

}  // namespace pt
