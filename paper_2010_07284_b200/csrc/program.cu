// program.cu -- device-resident evaluation of a whole task DAG.
//
// Replaces the reference executor's per-node scheduling (executor::run,
// proj/src/executor.cpp:117-282: a ready queue on a CPU WorkerPool that keeps
// every node's Value alive until the end, executor.cpp:119-123) with:
//
//  1. type inference over the Task list (task_graph.hpp:20-24, ids are a
//     topological order, task_graph.cpp:64-70) with the evalTask checks and
//     messages (executor.cpp:29-115); a failing task aborts its dependents
//     while independent branches still run (executor.cpp:178-218);
//  2. lowering to device steps with fusion: chains of thresholds and ! & |
//     become one fused launch (fused.cu); near(near(..)) runs become one
//     near_k launch; near(!e) becomes !interior(e) (one erosion launch);
//  3. liveness-based memory planning into one arena (an image's buffer is
//     reused as soon as its last consumer ran);
//  4. capture of the whole step list into a CUDA graph, replayed per run.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <sstream>

#include "slcs_internal.h"

namespace slcs {
slcs_image* new_image(slcs_ctx* ctx, int kind, int w, int h, int batch);
void drop_image(slcs_image* img);
void threshold_interval(int op, double n, int& lo, int& hi);
}  // namespace slcs

using namespace slcs;

namespace {

template <class F>
int pguard(F&& f) {
  try {
    f();
    const cudaError_t e = cudaGetLastError();  // launch errors of this call (per thread)
    if (e != cudaSuccess) {
      set_last_error(std::string("CUDA error: ") + cudaGetErrorString(e));
      return e == cudaErrorMemoryAllocation ? SLCS_ERR_OOM : SLCS_ERR_CUDA;
    }
    return SLCS_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    cudaGetLastError();
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SLCS_ERR_RUN;
  }
}

enum Op {
  OP_CONST, OP_LOAD, OP_SAVE, OP_PRINT, OP_INTENSITY, OP_NEAR, OP_NOT, OP_AND, OP_OR, OP_REACH,
  OP_THRESH, OP_ARITH, OP_VOLUME, OP_MAXVOL, OP_COMPONENTS
};

struct PTask {
  Op op;
  int sub = 0;
  double num = 0;
  std::string str, opcode;
  std::vector<int> deps;
};

enum VT { VT_NONE = 0, VT_NUM, VT_BOOL, VT_U16, VT_LABEL, VT_AUX };

const char* vt_name(VT t) {
  switch (t) {
    case VT_BOOL: return "bool";
    case VT_U16: return "u16";
    case VT_LABEL: return "label";
    default: return "number";
  }
}

// elementwise expression pool (trees over materialised leaves)
enum EK { E_LEAF, E_THRESH, E_NOT, E_AND, E_OR };
struct Expr {
  EK k;
  int a = -1, b = -1;  // child expr ids
  int lg = -1;         // leaf LG node (bool for E_LEAF, u16 for E_THRESH)
  int lo = 0, hi = 0;
  int ops = 1;         // op count of the subtree
  int need = 1;        // Sethi-Ullman register need
};

enum LK { LG_INPUT, LG_EW, LG_NEAR, LG_REACH, LG_MAXVOL, LG_VOLUME, LG_ARITH, LG_THRESH_DEV,
          LG_LABELS, LG_CCL };

struct LG {
  LK kind;
  VT type = VT_BOOL;
  int w = 0, h = 0, batch = 1;
  std::vector<int> in;  // LG inputs (images)
  int expr = -1;        // LG_EW root expression
  int k = 1;
  int tk = 0;  // LG_REACH: the target operand is near^tk(in[0]); k = 0 emits the selection
  bool erode = false;
  int cmp = 0;
  char aop = '+';
  int num_out = -1, num_a = -1, num_b = -1;
  double ca = 0, cb = 0;
  int gen_idx = -1;  // LG_REACH against an LG_LABELS input (label CSE)
  // label-CSE reach chain in one persistent launch (k_reach_chain): this node is
  // the last of chain_len reaches; in[0] is the first one's target, the
  // intermediate reaches close with near^chain_kmid, this one with near^k
  int chain_len = 1, chain_kmid = 0, chain_idx0 = -1;
  std::string name;  // LG_INPUT
  bool dead = false, output = false;
  int group = -1;  // leader of its shared launch (EW siblings, batched small reaches)
  int pro_expr = -1, epi_expr = -1, epi_src = -1;  // small maxvol: folded listings
  int consumers = 0, last_use = -1;
  size_t bytes = 0, offset = 0;
  void* ptr = nullptr;
};

struct Val {
  VT type = VT_NONE;
  int w = 0, h = 0, batch = 1;
  bool host_num = false;
  double num = 0;
  int numslot = -1;
  int lg = -1;        // materialised LG node
  int expr = -1;      // pending elementwise expression (not yet materialised)
  std::string err;    // set when the task failed or was aborted
  bool aborted = false;
};

struct InputSlot {
  int kind = -1, w = 0, h = 0, batch = 0;
  Geo geo;
  void* data = nullptr;
  size_t bytes = 0;
  const slcs_image* bound = nullptr;
  const slcs_image* copied = nullptr;  // bound image whose bytes are already in `data`
  bool host_set = false;
};

int op_arity(Op op) {
  switch (op) {
    case OP_CONST:
    case OP_LOAD: return 0;
    case OP_AND:
    case OP_OR:
    case OP_REACH:
    case OP_THRESH:
    case OP_ARITH: return 2;
    default: return 1;
  }
}

bool parse_opcode(const std::string& s, Op& op, int& sub) {
  static const std::map<std::string, std::pair<Op, int>> table = {
      {"const", {OP_CONST, 0}},   {"load", {OP_LOAD, 0}},     {"save", {OP_SAVE, 0}},
      {"print", {OP_PRINT, 0}},   {"intensity", {OP_INTENSITY, 0}},
      {"near", {OP_NEAR, 0}},     {"!", {OP_NOT, 0}},         {"&", {OP_AND, 0}},
      {"|", {OP_OR, 0}},          {"reach", {OP_REACH, 0}},   {">.", {OP_THRESH, SLCS_GT}},
      {">=.", {OP_THRESH, SLCS_GE}}, {"<.", {OP_THRESH, SLCS_LT}},
      {"<=.", {OP_THRESH, SLCS_LE}}, {"=.", {OP_THRESH, SLCS_EQ}},
      {"+", {OP_ARITH, '+'}},     {"-", {OP_ARITH, '-'}},     {"*", {OP_ARITH, '*'}},
      {"/", {OP_ARITH, '/'}},     {"volume", {OP_VOLUME, 0}}, {"maxvol", {OP_MAXVOL, 0}},
      {"components", {OP_COMPONENTS, 0}},
  };
  auto it = table.find(s);
  if (it == table.end()) return false;
  op = it->second.first;
  sub = it->second.second;
  return true;
}

size_t unit_of(VT t) { return t == VT_U16 ? 2 : 4; }

Geo geo_of(VT t, int w, int h, int b) {
  if (t == VT_U16) return u16_geo(w, h, b);
  if (t == VT_LABEL) return label_geo(w, h, b);
  return bool_geo(w, h, b);
}

// device scalar arithmetic: out = a op b; division by zero raises a flag
__global__ void k_arith(const double* nums, int a, int b, double ca, double cb, int out, char op,
                        int* err, int err_code) {
  slcs_pdl_wait();
  double x = a >= 0 ? nums[a] : ca;
  double y = b >= 0 ? nums[b] : cb;
  double r = 0;
  switch (op) {
    case '+': r = x + y; break;
    case '-': r = x - y; break;
    case '*': r = x * y; break;
    default:
      if (y == 0.0) {
        atomicCAS(err, 0, err_code);
        r = 0;
      } else {
        r = x / y;
      }
  }
  // x86-64 SSE NaN rules, so prints match the reference bit for bit ("-nan" vs
  // "nan" under %.6g): an invalid operation (inf - inf, 0 * inf) yields the
  // default NaN, which has the sign bit set; a NaN operand propagates (the
  // first one when both are NaN).  The GPU's own default NaN is positive.
  if (r != r) {
    const unsigned long long q = 0x0008000000000000ull;
    if (x != x) r = __longlong_as_double(__double_as_longlong(x) | q);
    else if (y != y) r = __longlong_as_double(__double_as_longlong(y) | q);
    else r = __longlong_as_double(0xfff8000000000000ull);
  }
  const_cast<double*>(nums)[out] = r;
}

}  // namespace

struct slcs_program {
  slcs_ctx* ctx = nullptr;
  // Guards this program's state.  A program runs on its own stream and touches
  // the context only through thread-safe calls (stream-ordered allocation,
  // event record/wait, the atomic launch counter), so its synchronisations
  // (division-by-zero check, downloads) never hold the context lock.
  std::mutex mu;
  std::vector<PTask> tasks;
  std::map<std::string, InputSlot> inputs;

  // plan state
  bool planned = false;
  int planned_fusion = -1;
  std::vector<Val> vals;
  std::vector<LG> lgs;
  std::vector<Expr> exprs;
  int n_nums = 0;
  int first_fail = -1;
  std::string fail_msg;
  void* arena = nullptr;
  size_t arena_bytes = 0;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  double* d_nums = nullptr;
  unsigned long long* d_counts = nullptr;
  int* d_err = nullptr;
  bool label_cse_used = false;
  void* staging = nullptr;
  size_t staging_bytes = 0;
  bool has_dev_arith = false;

  cudaStream_t pstream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int launches_per_run = 0;
  std::string plan_text;
  std::vector<int> exec_order;  // live steps in launch order (after reordering)
  // per-step device timeline (flag 16, observability): one event before the first
  // step and one after each step; tl_step[q] = index of LG q's interval
  bool timeline = false;
  std::vector<cudaEvent_t> tl_ev;
  std::vector<int> tl_step;
  std::vector<float> tl_ms;  // [2*i] start, [2*i+1] end of interval i (ms from the start)

  ~slcs_program() {
    release_plan();
    for (cudaEvent_t e : tl_ev) cudaEventDestroy(e);
  }

  cudaEvent_t tl_event(size_t i) {
    while (tl_ev.size() <= i) {
      cudaEvent_t e;
      cuda_check(cudaEventCreate(&e), "timeline event");
      tl_ev.push_back(e);
    }
    return tl_ev[i];
  }

  void release_plan() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
    if (arena) cudaFree(arena);
    if (scratch) cudaFree(scratch);
    if (d_nums) cudaFree(d_nums);
    if (d_counts) cudaFree(d_counts);
    if (d_err) cudaFree(d_err);
    arena = scratch = nullptr;
    d_nums = nullptr;
    d_counts = nullptr;
    d_err = nullptr;
    planned = false;
  }

  // ---------------------------------------------------------------- planning
  int add_lg(LG n) {
    lgs.push_back(std::move(n));
    return int(lgs.size()) - 1;
  }
  int add_expr(Expr e) {
    exprs.push_back(e);
    return int(exprs.size()) - 1;
  }

  int leaf(int lg) {
    Expr e;
    e.k = E_LEAF;
    e.lg = lg;
    return add_expr(e);
  }

  // number of distinct leaves of each kind in an expression
  void leaves(int e, std::vector<int>& b, std::vector<int>& u) const {
    const Expr& x = exprs[e];
    if (x.k == E_LEAF) {
      if (std::find(b.begin(), b.end(), x.lg) == b.end()) b.push_back(x.lg);
    } else if (x.k == E_THRESH) {
      if (std::find(u.begin(), u.end(), x.lg) == u.end()) u.push_back(x.lg);
    } else {
      leaves(x.a, b, u);
      if (x.b >= 0) leaves(x.b, b, u);
    }
  }

  bool fits(int e) const {
    std::vector<int> b, u;
    leaves(e, b, u);
    return exprs[e].ops + 2 <= kFusedMaxOps && exprs[e].need <= kFusedRegs &&
           int(b.size()) <= kFusedMaxIn && int(u.size()) <= kFusedMaxIn;
  }

  // the steps of the launch group led by `lead`, in launch order; `bad` when an
  // input of any member has no storage
  std::vector<int> group_members(int lead, bool& bad) const {
    std::vector<int> m;
    for (int q : exec_order)
      if (q == lead || lgs[q].group == lead) {
        if (q != lead && lgs[q].group != lead) continue;
        for (int i : lgs[q].in)
          if (!lgs[i].ptr) bad = true;
        m.push_back(q);
      }
    return m;
  }

  bool bool_only(int e) const {
    const Expr& x = exprs[e];
    if (x.k == E_THRESH) return false;
    if (x.k == E_LEAF) return true;
    return bool_only(x.a) && (x.b < 0 || bool_only(x.b));
  }

  // a one-output listing for a folded prologue/epilogue (preset_lg's value is
  // the host kernel's own result word)
  FusedProgram listing(int e, int preset_lg) {
    FusedProgram fp;
    std::vector<const uint32_t*> bin;
    std::vector<const uint16_t*> uin;
    fwd_.clear();
    if (preset_lg >= 0) fwd_[preset_lg] = -1;
    const int r = compile_expr(e, fp, bin, uin, 0);
    fwd_.clear();
    FusedOp st_op;
    st_op.op = FOP_STORE;
    st_op.dst = uint8_t(r);
    st_op.a = st_op.b = 0;
    st_op.lo = st_op.hi = 0;
    fp.ops[fp.n_ops++] = st_op;
    for (size_t z = 0; z < bin.size(); ++z) fp.bin[z] = bin[z];
    fp.n_bin = int(bin.size());
    return fp;
  }

  // can these LG_EW steps (in order) run as one multi-output listing?
  bool group_fits(const std::vector<int>& grp) const {
    std::vector<int> b, u;
    int ops = 0, need = 0, saved = 0;
    for (size_t i = 0; i < grp.size(); ++i) {
      const int e = lgs[grp[i]].expr;
      leaves(e, b, u);
      ops += exprs[e].ops + 1;  // + its store
      need = std::max(need, exprs[e].need);
      for (size_t k = i + 1; k < grp.size(); ++k)  // read by a later member: forwarded
        if (std::find(lgs[grp[k]].in.begin(), lgs[grp[k]].in.end(), grp[i]) !=
            lgs[grp[k]].in.end()) {
          ++saved;
          ++ops;  // the copy into its saved register
          break;
        }
    }
    int nb = 0;  // bool leaves that are not members (members are forwarded)
    for (int q : b)
      if (std::find(grp.begin(), grp.end(), q) == grp.end()) ++nb;
    return ops <= kFusedMaxOps && need + saved <= kFusedRegs && nb <= kFusedMaxIn &&
           int(u.size()) <= kFusedMaxIn;
  }

  // materialise a pending expression as an LG_EW node (or return its leaf)
  int materialize_expr(int e, int w, int h, int b) {
    if (exprs[e].k == E_LEAF) return exprs[e].lg;
    LG n;
    n.kind = LG_EW;
    n.type = VT_BOOL;
    n.w = w;
    n.h = h;
    n.batch = b;
    n.expr = e;
    std::vector<int> bl, ul;
    leaves(e, bl, ul);
    n.in = bl;
    n.in.insert(n.in.end(), ul.begin(), ul.end());
    return add_lg(n);
  }

  int materialize(Val& v) {
    if (v.lg < 0) {
      v.lg = materialize_expr(v.expr, v.w, v.h, v.batch);
      v.expr = -1;
    }
    return v.lg;
  }

  // pending expression view of a bool/u16 value used as a boolean operand
  int as_expr(Val& v, bool fusion, bool shared = false) {
    if (v.expr >= 0) {
      // an expression with several consumers is materialised once rather
      // than recomputed (re-reading u16 pixels costs 16x the bit image)
      if (!fusion || shared) materialize(v);
      else return v.expr;
    }
    if (v.type == VT_U16) {  // boolArg coercion p > 0 (executor.cpp:43-50)
      Expr e;
      e.k = E_THRESH;
      e.lg = v.lg;
      e.lo = 1;
      e.hi = 65535;
      return add_expr(e);
    }
    return leaf(v.lg);
  }

  int make_unary_not(int a) {
    if (exprs[a].k == E_NOT) return exprs[a].a;  // !!e = e
    Expr e;
    e.k = E_NOT;
    e.a = a;
    e.ops = exprs[a].ops + 1;
    e.need = exprs[a].need;
    return add_expr(e);
  }

  int make_binary(EK k, int a, int b) {
    Expr e;
    e.k = k;
    e.a = a;
    e.b = b;
    e.ops = exprs[a].ops + exprs[b].ops + 1;
    int na = exprs[a].need, nb = exprs[b].need;
    e.need = na == nb ? na + 1 : std::max(na, nb);
    return add_expr(e);
  }

  void plan(int fusion, bool label_cse, bool chain) {
    release_plan();
    vals.assign(tasks.size(), Val{});
    lgs.clear();
    exprs.clear();
    n_nums = 0;
    first_fail = -1;
    fail_msg.clear();
    has_dev_arith = false;
    const bool fuse = fusion != 0;

    // consumers per task (aliases intensity/save/print resolved later)
    std::vector<int> consumers(tasks.size(), 0);
    std::vector<bool> is_output(tasks.size(), false);
    for (size_t i = 0; i < tasks.size(); ++i) {
      for (int d : tasks[i].deps) consumers[d]++;
      if (tasks[i].op == OP_SAVE || tasks[i].op == OP_PRINT) is_output[i] = true;
    }
    // effective consumers of the storage behind aliases
    std::vector<int> eff = consumers;
    std::vector<bool> eff_out(tasks.size(), false);
    for (int i = int(tasks.size()) - 1; i >= 0; --i) {
      const PTask& t = tasks[i];
      if (t.op == OP_INTENSITY || t.op == OP_SAVE || t.op == OP_PRINT) {
        int d = t.deps[0];
        eff[d] += eff[i] - 1 + (t.op != OP_INTENSITY ? 1 : 0);
        if (t.op != OP_INTENSITY || eff_out[i]) eff_out[d] = true;
      }
    }

    // reaches per `through` task: a labelling shared by >= 2 reaches is
    // computed once (label CSE) when enabled
    std::vector<int> reach_uses(tasks.size(), 0);
    for (const PTask& t : tasks)
      if (t.op == OP_REACH) reach_uses[t.deps[1]]++;
    std::map<int, int> labels_of;  // through LG -> LG_LABELS
    int labeled = 0;
    label_cse_used = false;

    auto fail_task = [&](int i, const std::string& msg) {
      vals[i].err = msg;
      if (first_fail < 0) {
        first_fail = i;
        fail_msg = "task " + std::to_string(i) + " (" + tasks[i].opcode + ") failed: " + msg;
      }
    };

    for (size_t ii = 0; ii < tasks.size(); ++ii) {
      const int i = int(ii);
      const PTask& t = tasks[i];
      Val& v = vals[i];
      bool aborted = false;
      for (int d : t.deps)
        if (!vals[d].err.empty()) aborted = true;
      if (aborted) {
        v.err = "aborted";
        v.aborted = true;
        continue;
      }
      auto img_arg = [&](int d) -> Val& {
        Val& x = vals[d];
        if (x.type == VT_NUM)
          throw Error(SLCS_ERR_KIND, "'" + t.opcode + "' expects an image, got a number");
        return x;
      };
      auto bool_arg = [&](int d) -> Val& {
        Val& x = img_arg(d);
        if (x.type == VT_LABEL)
          throw Error(SLCS_ERR_KIND, "'" + t.opcode + "' expects a boolean image, got label");
        return x;
      };
      auto num_arg = [&](int d) -> Val& {
        Val& x = vals[d];
        if (x.type != VT_NUM) {
          std::string desc = "image(" + std::to_string(x.w) + "x" + std::to_string(x.h) + "," +
                             vt_name(x.type) + ")";
          throw Error(SLCS_ERR_KIND, "'" + t.opcode + "' expects a number, got " + desc);
        }
        return x;
      };
      auto same = [&](const Val& a, const Val& b, const char* what) {
        if (a.w != b.w || a.h != b.h || a.batch != b.batch)
          throw Error(SLCS_ERR_SHAPE, std::string(what) + ": dimension mismatch (" +
                                          std::to_string(a.w) + "x" + std::to_string(a.h) +
                                          " vs " + std::to_string(b.w) + "x" +
                                          std::to_string(b.h) + ")");
      };
      auto shape_from = [&](const Val& a) {
        v.w = a.w;
        v.h = a.h;
        v.batch = a.batch;
      };
      try {
        switch (t.op) {
          case OP_CONST:
            v.type = VT_NUM;
            v.host_num = true;
            v.num = t.num;
            break;
          case OP_LOAD: {
            auto it = inputs.find(t.str);
            if (it == inputs.end() || it->second.kind < 0)
              throw Error(SLCS_ERR_RUN, "cannot open file for reading: " + t.str);
            const InputSlot& s = it->second;
            v.type = s.kind == SLCS_U16 ? VT_U16 : (s.kind == SLCS_LABEL ? VT_LABEL : VT_BOOL);
            v.w = s.w;
            v.h = s.h;
            v.batch = s.batch;
            // one LG_INPUT per distinct name
            int found = -1;
            for (size_t q = 0; q < lgs.size(); ++q)
              if (lgs[q].kind == LG_INPUT && lgs[q].name == t.str) found = int(q);
            if (found < 0) {
              LG n;
              n.kind = LG_INPUT;
              n.type = v.type;
              n.w = v.w;
              n.h = v.h;
              n.batch = v.batch;
              n.name = t.str;
              found = add_lg(n);
            }
            v.lg = found;
            break;
          }
          case OP_SAVE: {
            Val& x = vals[t.deps[0]];
            if (x.type == VT_NUM)
              throw Error(SLCS_ERR_RUN, "cannot save a number as an image (use print)");
            v = x;
            materialize(vals[t.deps[0]]);
            v = vals[t.deps[0]];
            lgs[v.lg].output = true;
            break;
          }
          case OP_PRINT: {
            Val& x = vals[t.deps[0]];
            if (x.type != VT_NUM) {
              materialize(x);
              lgs[x.lg].output = true;
            }
            v = x;
            break;
          }
          case OP_INTENSITY: {
            Val& x = img_arg(t.deps[0]);
            if (x.type != VT_U16)
              throw Error(SLCS_ERR_KIND, std::string("'intensity' expects a numeric image, got ") +
                                             vt_name(x.type));
            v = x;
            break;
          }
          case OP_THRESH: {
            Val& x = img_arg(t.deps[0]);
            Val& n = num_arg(t.deps[1]);
            const char* sym[] = {">.", ">=.", "<.", "<=.", "=."};
            if (x.type != VT_U16)
              throw Error(SLCS_ERR_KIND, std::string(sym[t.sub]) + " expects a numeric image, got " +
                                             vt_name(x.type));
            v.type = VT_BOOL;
            shape_from(x);
            if (n.host_num) {
              Expr e;
              e.k = E_THRESH;
              e.lg = x.lg;
              threshold_interval(t.sub, n.num, e.lo, e.hi);
              v.expr = add_expr(e);
            } else {
              LG g;
              g.kind = LG_THRESH_DEV;
              g.w = x.w;
              g.h = x.h;
              g.batch = x.batch;
              g.in = {x.lg};
              g.cmp = t.sub;
              g.num_a = n.numslot;
              v.lg = add_lg(g);
            }
            break;
          }
          case OP_NOT: {
            Val& x = bool_arg(t.deps[0]);
            v.type = VT_BOOL;
            shape_from(x);
            v.expr = make_unary_not(as_expr(x, fuse, eff[t.deps[0]] > 1));
            break;
          }
          case OP_AND:
          case OP_OR: {
            Val& x = bool_arg(t.deps[0]);
            Val& y = bool_arg(t.deps[1]);
            same(x, y, t.opcode.c_str());
            v.type = VT_BOOL;
            shape_from(x);
            int a = as_expr(x, fuse, eff[t.deps[0]] > 1), b = as_expr(y, fuse, eff[t.deps[1]] > 1);
            int e = make_binary(t.op == OP_AND ? E_AND : E_OR, a, b);
            if (!fits(e)) {
              // keep launches bounded: materialise the operands first
              int la = materialize_expr(a, x.w, x.h, x.batch);
              int lb = materialize_expr(b, y.w, y.h, y.batch);
              e = make_binary(t.op == OP_AND ? E_AND : E_OR, leaf(la), leaf(lb));
            }
            v.expr = e;
            break;
          }
          case OP_NEAR: {
            Val& x = bool_arg(t.deps[0]);
            v.type = VT_BOOL;
            shape_from(x);
            // near(!e) = !interior(e)  (De Morgan on the clipped window)
            if (fuse && x.expr >= 0 && exprs[x.expr].k == E_NOT && eff[t.deps[0]] == 1 &&
                !eff_out[t.deps[0]]) {
              int inner = exprs[x.expr].a;
              LG g;
              g.kind = LG_NEAR;
              g.erode = true;
              g.w = x.w;
              g.h = x.h;
              g.batch = x.batch;
              g.in = {materialize_expr(inner, x.w, x.h, x.batch)};
              int lg = add_lg(g);
              v.expr = make_unary_not(leaf(lg));
            } else {
              int src = x.type == VT_U16 ? materialize_expr(as_expr(x, fuse), x.w, x.h, x.batch)
                                         : materialize(x);
              LG g;
              g.kind = LG_NEAR;
              g.w = x.w;
              g.h = x.h;
              g.batch = x.batch;
              g.in = {src};
              v.lg = add_lg(g);
            }
            break;
          }
          case OP_REACH: {
            Val& x = bool_arg(t.deps[0]);
            Val& y = bool_arg(t.deps[1]);
            if (x.w != y.w || x.h != y.h || x.batch != y.batch)
              throw Error(SLCS_ERR_SHAPE, "reach: dimension mismatch (" + std::to_string(x.w) +
                                              "x" + std::to_string(x.h) + " vs " +
                                              std::to_string(y.w) + "x" + std::to_string(y.h) +
                                              ")");
            v.type = VT_BOOL;
            shape_from(x);
            int a = x.type == VT_U16 ? materialize_expr(as_expr(x, fuse), x.w, x.h, x.batch)
                                     : materialize(x);
            int b = y.type == VT_U16 ? materialize_expr(as_expr(y, fuse), y.w, y.h, y.batch)
                                     : materialize(y);
            LG g;
            g.kind = LG_REACH;
            g.w = x.w;
            g.h = x.h;
            g.batch = x.batch;
            g.in = {a, b};
            if (label_cse && reach_uses[t.deps[1]] >= 2 && !ccl_small_path(x.w, x.h) &&
                labeled < 4096) {
              auto it = labels_of.find(b);
              if (it == labels_of.end()) {
                LG l;
                l.kind = LG_LABELS;
                l.type = VT_AUX;
                l.w = x.w;
                l.h = x.h;
                l.batch = x.batch;
                l.in = {b};
                it = labels_of.emplace(b, add_lg(l)).first;
              }
              g.in.push_back(it->second);
              g.gen_idx = labeled++;
              label_cse_used = true;
            }
            v.lg = add_lg(g);
            break;
          }
          case OP_COMPONENTS: {
            // components(x): the canonical ccl::label image (ccl.hpp:52-60) as a
            // value -- new, like maxvol; label images are saved as RGB (png_io)
            Val& x = bool_arg(t.deps[0]);
            int a = x.type == VT_U16 ? materialize_expr(as_expr(x, fuse), x.w, x.h, x.batch)
                                     : materialize(x);
            if ((unsigned long long)x.w * (unsigned long long)x.h >= 0xfffffffeull)
              throw Error(SLCS_ERR_TOO_LARGE, "image too large for packed coordinate labels");
            LG g;
            g.kind = LG_CCL;
            g.type = VT_LABEL;
            g.w = x.w;
            g.h = x.h;
            g.batch = x.batch;
            g.in = {a};
            v.type = VT_LABEL;
            shape_from(x);
            v.lg = add_lg(g);
            break;
          }
          case OP_MAXVOL:
          case OP_VOLUME: {
            Val& x = bool_arg(t.deps[0]);
            int a = x.type == VT_U16 ? materialize_expr(as_expr(x, fuse), x.w, x.h, x.batch)
                                     : materialize(x);
            LG g;
            g.kind = t.op == OP_VOLUME ? LG_VOLUME : LG_MAXVOL;
            g.w = x.w;
            g.h = x.h;
            g.batch = x.batch;
            g.in = {a};
            if (t.op == OP_VOLUME) {
              v.type = VT_NUM;
              g.type = VT_NUM;
              g.num_out = v.numslot = n_nums;
              n_nums += x.batch;
            } else {
              v.type = VT_BOOL;
              shape_from(x);
            }
            v.lg = add_lg(g);
            break;
          }
          case OP_ARITH: {
            Val& x = num_arg(t.deps[0]);
            Val& y = num_arg(t.deps[1]);
            v.type = VT_NUM;
            if (x.host_num && y.host_num) {
              double r = 0;
              switch (t.sub) {
                case '+': r = x.num + y.num; break;
                case '-': r = x.num - y.num; break;
                case '*': r = x.num * y.num; break;
                default:
                  if (y.num == 0.0) throw Error(SLCS_ERR_RUN, "division by zero");
                  r = x.num / y.num;
              }
              v.host_num = true;
              v.num = r;
            } else {
              LG g;
              g.kind = LG_ARITH;
              g.type = VT_NUM;
              g.aop = char(t.sub);
              g.num_a = x.host_num ? -1 : x.numslot;
              g.num_b = y.host_num ? -1 : y.numslot;
              g.ca = x.num;
              g.cb = y.num;
              g.num_out = v.numslot = n_nums++;
              // remember the task id for error reporting
              g.k = i;
              v.lg = add_lg(g);
              has_dev_arith = true;
            }
            break;
          }
        }
      } catch (const Error& e) {
        fail_task(i, e.what());
      }
    }

    // ---- near-chain merging: near^a(near^b(x)) -> near^(a+b)(x), k <= 8
    for (LG& n : lgs) n.consumers = 0;
    for (const LG& n : lgs)
      for (int q : n.in) lgs[q].consumers++;
    if (fuse) {
      for (size_t q = 0; q < lgs.size(); ++q) {
        LG& n = lgs[q];
        if (n.kind != LG_NEAR || n.dead) continue;
        for (;;) {
          LG& m = lgs[n.in[0]];
          if (m.kind != LG_NEAR || m.erode != n.erode || m.consumers != 1 || m.output ||
              n.k + m.k > 8)
            break;
          n.k += m.k;
          n.in[0] = m.in[0];
          m.dead = true;
        }
        // near(reach(t, u)): reach closes with near(t | S), so a following
        // near widens that closing stencil instead of running separately
        LG& m = lgs[n.in[0]];
        if (!n.erode && m.kind == LG_REACH && m.consumers == 1 && !m.output &&
            !ccl_small_path(m.w, m.h) && n.k + m.k <= 8) {
          const int k = n.k + m.k;
          const bool out = n.output;
          LG merged = m;
          merged.k = k;
          merged.output = out;
          m.dead = true;
          n = merged;
        }
      }
    }

    // ---- nears folded into reach targets: the fused reach stages its target
    // window with a wider halo and applies near^tk itself (tk <= 2), and a
    // reach whose only consumer is another reach's target emits its selection
    // t | S (k = 0) -- the consumer applies the closing near^k as part of its tk.
    // The chain near -> reach -> near -> reach ... becomes one launch per reach.
    if (fuse) {
      for (LG& n : lgs) n.consumers = 0;
      for (const LG& n : lgs)
        if (!n.dead)
          for (int q : n.in) lgs[q].consumers++;
      for (LG& n : lgs) {
        if (n.dead || n.kind != LG_REACH || n.gen_idx >= 0 || ccl_small_path(n.w, n.h)) continue;
        LG& m = lgs[n.in[0]];
        if (m.kind == LG_NEAR && !m.erode && m.consumers == 1 && !m.output &&
            n.tk + m.k <= 2) {
          n.tk += m.k;
          n.in[0] = m.in[0];
          m.dead = true;
        } else if (m.kind == LG_REACH && !m.dead && m.gen_idx < 0 && m.consumers == 1 &&
                   !m.output && m.k >= 1 && n.tk + m.k <= 2 && m.w == n.w && m.h == n.h &&
                   m.batch == n.batch && n.in[1] != n.in[0]) {
          n.tk += m.k;
          m.k = 0;
        }
      }
    }

    // ---- chains of label-CSE reaches (same labelling, each the next one's only
    // input) run as ONE persistent cooperative launch (k_reach_chain) when the
    // tile grid is co-resident: the config-2 chain's 500 reaches become 1 launch
    if (fuse && label_cse && chain) {
      for (LG& n : lgs) n.consumers = 0;
      for (const LG& n : lgs)
        if (!n.dead)
          for (int q : n.in) lgs[q].consumers++;
      for (LG& n : lgs) {
        if (n.dead || n.kind != LG_REACH || n.gen_idx < 0) continue;
        if (n.chain_idx0 < 0) n.chain_idx0 = n.gen_idx;
        LG& m = lgs[n.in[0]];
        if (m.dead || m.kind != LG_REACH || m.gen_idx < 0 || m.consumers != 1 || m.output ||
            m.in[1] != n.in[1] || m.in[2] != n.in[2] || m.k > 2 ||
            (m.chain_len > 1 && m.chain_kmid != m.k) || m.w != n.w || m.h != n.h ||
            m.batch != n.batch)
          continue;
        const int idx0 = m.chain_idx0 < 0 ? m.gen_idx : m.chain_idx0;
        if (n.gen_idx != idx0 + m.chain_len) continue;
        if (!reach_chain_fits(bool_geo(n.w, n.h, n.batch), m.chain_len + 1, m.k,
                              std::max(1, n.k)))
          continue;
        n.chain_len = m.chain_len + 1;
        n.chain_kmid = m.k;
        n.chain_idx0 = idx0;
        n.in[0] = m.in[0];
        m.dead = true;
      }
    }

    // ---- small-image maxvol absorbs a bool-only elementwise operand (prologue)
    // and a bool-only elementwise consumer (epilogue): k_small evaluates them
    // per word, so grow -> maxvol -> "| surrounded" (C3) is one launch
    if (fuse) {
      auto recount = [&] {
        for (LG& n : lgs) n.consumers = 0;
        for (const LG& n : lgs)
          if (!n.dead)
            for (int q : n.in) lgs[q].consumers++;
      };
      auto same_shape = [](const LG& a, const LG& b) {
        return a.w == b.w && a.h == b.h && a.batch == b.batch;
      };
      recount();
      for (LG& n : lgs) {
        if (n.dead || n.kind != LG_MAXVOL || !ccl_small_path(n.w, n.h)) continue;
        LG& m = lgs[n.in[0]];
        if (m.kind == LG_EW && !m.dead && m.consumers == 1 && !m.output && bool_only(m.expr) &&
            same_shape(m, n)) {
          n.pro_expr = m.expr;
          n.in = m.in;
          m.dead = true;
        }
      }
      recount();
      for (size_t q = 0; q < lgs.size(); ++q) {
        LG& e = lgs[q];
        if (e.dead || e.kind != LG_EW || !bool_only(e.expr)) continue;
        const std::vector<int> ins = e.in;  // e is overwritten below
        for (int i : ins) {
          LG& m = lgs[i];
          if (m.kind != LG_MAXVOL || m.dead || m.consumers != 1 || m.output || m.epi_expr >= 0 ||
              !ccl_small_path(m.w, m.h) || !same_shape(m, e))
            continue;
          // e becomes the maxvol step, its own expression the epilogue (values
          // refer to e's index, so e keeps it)
          LG nm = m;
          nm.epi_expr = e.expr;
          nm.epi_src = i;
          nm.output = e.output;
          for (int z : e.in)
            if (z != i && std::find(nm.in.begin(), nm.in.end(), z) == nm.in.end())
              nm.in.push_back(z);
          m.dead = true;
          e = nm;
          break;
        }
      }
    }

    std::vector<int> order;
    for (size_t q = 0; q < lgs.size(); ++q)
      if (!lgs[q].dead && lgs[q].kind != LG_INPUT) order.push_back(int(q));

    // ---- reorder (list scheduling): among the ready steps, prefer one that can
    // share a launch with the step just scheduled (an elementwise sibling, or an
    // independent small reach of the same shape), else the earliest.  The
    // reference runs independent nodes concurrently (executor.cpp:220, 259); here
    // they share launches instead.
    auto small_reach = [&](const LG& n) {
      return n.kind == LG_REACH && n.gen_idx < 0 && n.k == 1 && n.tk == 0 &&
             ccl_small_path(n.w, n.h);
    };
    auto joinable = [&](const LG& a, const LG& b) {
      if (a.w != b.w || a.h != b.h || a.batch != b.batch) return false;
      return (a.kind == LG_EW && b.kind == LG_EW) || (small_reach(a) && small_reach(b));
    };
    if (fuse && order.size() > 2) {
      std::vector<char> done(lgs.size(), 0);
      for (size_t q = 0; q < lgs.size(); ++q)
        if (lgs[q].dead || lgs[q].kind == LG_INPUT) done[q] = 1;
      // device numbers are dependencies too (volume -> arith / threshold(dev))
      std::map<int, int> num_producer;
      for (size_t q = 0; q < lgs.size(); ++q)
        if (!lgs[q].dead && lgs[q].num_out >= 0) {
          const int nslots = lgs[q].kind == LG_VOLUME ? lgs[q].batch : 1;
          for (int z = 0; z < nslots; ++z) num_producer[lgs[q].num_out + z] = int(q);
        }
      auto num_ready = [&](int slot) {
        if (slot < 0) return true;
        auto it = num_producer.find(slot);
        return it == num_producer.end() || done[it->second];
      };
      std::vector<int> sched;
      std::vector<char> taken(order.size(), 0);
      while (sched.size() < order.size()) {
        int pick = -1;
        for (size_t i = 0; i < order.size(); ++i) {
          if (taken[i]) continue;
          const LG& c = lgs[order[i]];
          bool ready = num_ready(c.num_a) && num_ready(c.num_b);
          for (int in : c.in) ready = ready && done[in];
          if (!ready) continue;
          if (pick < 0) pick = int(i);
          if (!sched.empty() && joinable(lgs[sched.back()], lgs[order[i]])) {
            pick = int(i);
            break;
          }
        }
        if (pick < 0) break;  // (cannot happen for a DAG) keep the original order
        taken[pick] = 1;
        done[order[pick]] = 1;
        sched.push_back(order[pick]);
      }
      if (sched.size() == order.size()) order.swap(sched);
    }

    // ---- sibling merge: adjacent elementwise steps of one shape run as one
    // multi-output listing (a u16 image thresholded twice is read once, and a
    // member that a later member reads is forwarded in a register)
    for (LG& n : lgs) n.group = -1;
    if (fuse) {
      for (size_t i = 0; i < order.size();) {
        const LG& lead = lgs[order[i]];
        size_t j = i + 1;
        if (lead.kind == LG_EW) {
          std::vector<int> grp{order[i]};
          while (j < order.size() && int(grp.size()) < kFusedMaxOut) {
            const LG& c = lgs[order[j]];
            if (c.kind != LG_EW || c.w != lead.w || c.h != lead.h || c.batch != lead.batch)
              break;
            grp.push_back(order[j]);
            if (!group_fits(grp)) {
              grp.pop_back();
              break;
            }
            ++j;
          }
          if (grp.size() > 1)
            for (int q : grp) lgs[q].group = order[i];
        } else if (small_reach(lead)) {
          // independent small reaches of one shape: one k_small launch
          std::vector<int> grp{order[i]};
          while (j < order.size() && int(grp.size()) < 4 && small_reach(lgs[order[j]]) &&
                 joinable(lead, lgs[order[j]])) {
            bool dep = false;
            for (int q : grp)
              for (int in : lgs[order[j]].in) dep = dep || in == q;
            if (dep) break;
            grp.push_back(order[j]);
            ++j;
          }
          if (grp.size() > 1)
            for (int q : grp) lgs[q].group = order[i];
        } else if (lead.kind == LG_VOLUME && lead.batch == 1) {
          // adjacent volumes (independent: a volume reads an image, makes a
          // number): one k_volume_multi launch
          std::vector<int> grp{order[i]};
          while (j < order.size() && int(grp.size()) < kVolumeJobsMax &&
                 lgs[order[j]].kind == LG_VOLUME && lgs[order[j]].batch == 1) {
            grp.push_back(order[j]);
            ++j;
          }
          if (grp.size() > 1)
            for (int q : grp) lgs[q].group = order[i];
        }
        i = j;
      }
    }

    // ---- memory plan over live nodes in order; a sibling group is one step
    // (all its outputs are allocated before any of its inputs is recycled)
    std::vector<int> stepv(order.size());
    for (size_t pos = 0; pos < order.size(); ++pos) {
      const LG& n = lgs[order[pos]];
      stepv[pos] = (pos > 0 && n.group >= 0 && n.group != order[pos]) ? stepv[pos - 1] : int(pos);
    }
    for (LG& n : lgs) n.last_use = -1;
    for (size_t pos = 0; pos < order.size(); ++pos)
      for (int q : lgs[order[pos]].in) lgs[q].last_use = stepv[pos];
    struct Blk {
      size_t off, size;
    };
    std::vector<Blk> freel;
    size_t top = 0;
    auto alloc = [&](size_t bytes) -> size_t {
      bytes = round_up(bytes, 256);
      int best = -1;
      for (size_t f = 0; f < freel.size(); ++f)
        if (freel[f].size >= bytes && (best < 0 || freel[f].size < freel[best].size))
          best = int(f);
      if (best >= 0) {
        size_t off = freel[best].off;
        if (freel[best].size == bytes)
          freel.erase(freel.begin() + best);
        else {
          freel[best].off += bytes;
          freel[best].size -= bytes;
        }
        return off;
      }
      size_t off = top;
      top += bytes;
      return off;
    };
    auto release = [&](size_t off, size_t bytes) {
      bytes = round_up(bytes, 256);
      freel.push_back({off, bytes});
      std::sort(freel.begin(), freel.end(), [](const Blk& a, const Blk& b) { return a.off < b.off; });
      std::vector<Blk> merged;
      for (const Blk& b : freel) {
        if (!merged.empty() && merged.back().off + merged.back().size == b.off)
          merged.back().size += b.size;
        else
          merged.push_back(b);
      }
      freel.swap(merged);
    };
    size_t scratch_need = 0;
    for (size_t pos = 0; pos < order.size();) {
      size_t end = pos + 1;
      while (end < order.size() && stepv[end] == stepv[pos]) ++end;
      for (size_t p = pos; p < end; ++p) {
      LG& n = lgs[order[p]];
      if (n.type == VT_AUX) {
        // labelling + the reach flag stamps (one uint32 per 2x2 block, two copies:
        // a reach chain alternates them by step parity)
        n.bytes = round_up(ccl_labels_bytes(n.w, n.h, n.batch), 256) +
                  key_geo(n.w, n.h).slice_blocks * size_t(n.batch) * 4 * 2;
        n.offset = alloc(n.bytes);
      } else if (n.type != VT_NUM) {
        Geo g = geo_of(n.type, n.w, n.h, n.batch);
        n.bytes = g.slice * size_t(n.batch) * unit_of(n.type);
        n.offset = alloc(n.bytes);
      }
      if (n.kind == LG_REACH && n.gen_idx >= 0) {
        scratch_need = std::max(
            scratch_need, n.chain_len > 1
                              ? reach_chain_scratch_bytes(bool_geo(n.w, n.h, n.batch), n.chain_len)
                              : bool_geo(n.w, n.h, n.batch).slice * n.batch * 4);
      } else if (n.kind == LG_REACH) {
        size_t s = ccl_scratch_bytes(n.w, n.h, n.batch, true, false);
        if (!ccl_small_path(n.w, n.h)) s += bool_geo(n.w, n.h, n.batch).slice * n.batch * 4;
        scratch_need = std::max(scratch_need, s);
      } else if (n.kind == LG_MAXVOL || n.kind == LG_CCL) {
        scratch_need = std::max(scratch_need, ccl_scratch_bytes(n.w, n.h, n.batch, false, true));
      } else if (n.kind == LG_NEAR && n.k > 8) {
        scratch_need = std::max(scratch_need, n.bytes);
      }
      }
      // inputs whose last use is this step can be recycled now
      std::vector<int> uniq;
      for (size_t p = pos; p < end; ++p)
        uniq.insert(uniq.end(), lgs[order[p]].in.begin(), lgs[order[p]].in.end());
      std::sort(uniq.begin(), uniq.end());
      uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
      for (int q : uniq) {
        LG& m = lgs[q];
        if (m.kind != LG_INPUT && m.last_use == stepv[pos] && !m.output && m.type != VT_NUM)
          release(m.offset, m.bytes);
      }
      // a result nobody consumes (and not an output) is dead after its step
      for (size_t p = pos; p < end; ++p) {
        LG& n = lgs[order[p]];
        if (n.type != VT_NUM && n.last_use < 0 && !n.output) release(n.offset, n.bytes);
      }
      pos = end;
    }
    arena_bytes = top;
    scratch_bytes = scratch_need;
    exec_order = order;

    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (arena_bytes) cuda_check(cudaMalloc(&arena, arena_bytes), "program arena");
    if (scratch_bytes) cuda_check(cudaMalloc(&scratch, scratch_bytes), "program scratch");
    cuda_check(cudaMalloc(&d_nums, sizeof(double) * std::max(1, n_nums)), "program numbers");
    cuda_check(cudaMalloc(&d_counts, 2 * sizeof(unsigned long long) * std::max(1, n_nums)),
               "program counts");
    cuda_check(cudaMemset(d_counts, 0, 2 * sizeof(unsigned long long) * std::max(1, n_nums)),
               "program counts");
    cuda_check(cudaMalloc(&d_err, sizeof(int)), "program error flag");
    for (LG& n : lgs) {
      if (n.kind == LG_INPUT) n.ptr = inputs[n.name].data;
      else if (!n.dead && n.type != VT_NUM) n.ptr = static_cast<char*>(arena) + n.offset;
    }

    // ---- human-readable plan
    std::ostringstream os;
    os << "program: " << tasks.size() << " tasks -> " << order.size() << " device steps, arena "
       << arena_bytes << " B, scratch " << scratch_bytes << " B, fusion " << (fuse ? "on" : "off")
       << "\n";
    for (int q : order) {
      const LG& n = lgs[q];
      static const char* kn[] = {"input", "fused", "near", "reach", "maxvol", "volume", "arith",
                                 "threshold(dev)", "labels", "components"};
      os << "  step " << q << ": " << kn[n.kind];
      if (n.kind == LG_NEAR) os << (n.erode ? " interior" : " near") << "^" << n.k;
      if (n.kind == LG_EW) os << " (" << exprs[n.expr].ops << " ops)";
      if (n.pro_expr >= 0) os << " +prologue(" << exprs[n.pro_expr].ops << " ops)";
      if (n.epi_expr >= 0) os << " +epilogue(" << exprs[n.epi_expr].ops << " ops)";
      if (n.group >= 0)
        os << (n.group == q ? " [launch group lead]" : " [with step " + std::to_string(n.group) + "]");
      if (n.kind == LG_REACH && n.gen_idx >= 0) os << " (shared labelling)";
      if (n.kind == LG_REACH && n.chain_len > 1)
        os << " chain of " << n.chain_len << " reaches (one persistent launch, inner closing near^"
           << n.chain_kmid << ")";
      if (n.kind == LG_REACH && n.tk > 0) os << " target near^" << n.tk;
      if (n.kind == LG_REACH && n.k == 0) os << " emits selection";
      if (n.kind == LG_REACH && n.k > 1) os << " closing near^" << n.k;
      os << " " << n.w << "x" << n.h;
      if (n.batch > 1) os << "x" << n.batch;
      os << " in=[";
      for (size_t z = 0; z < n.in.size(); ++z) os << (z ? "," : "") << n.in[z];
      os << "]" << (n.output ? " output" : "") << "\n";
    }
    plan_text = os.str();
    planned = true;
  }

  // ------------------------------------------------------------------ emit
  std::map<int, int> fwd_;  // sibling LG -> register holding its value
  int compile_expr(int e, FusedProgram& fp, std::vector<const uint32_t*>& bin,
                   std::vector<const uint16_t*>& uin, int reg_base) {
    const Expr& x = exprs[e];
    auto add = [&](uint8_t op, int dst, int a, int b, int lo = 0, int hi = 0) {
      FusedOp o;
      o.op = op;
      o.dst = uint8_t(dst);
      o.a = uint8_t(a);
      o.b = uint8_t(b);
      o.lo = lo;
      o.hi = hi;
      fp.ops[fp.n_ops++] = o;
    };
    switch (x.k) {
      case E_LEAF: {
        auto f = fwd_.find(x.lg);
        if (f != fwd_.end() && f->second < 0) {  // the host kernel's result (epilogue)
          add(FOP_PRESET, reg_base, 0, 0);
          return reg_base;
        }
        if (f != fwd_.end()) {  // a sibling computed earlier in this listing
          add(FOP_OR, reg_base, f->second, f->second);
          return reg_base;
        }
        const uint32_t* p = static_cast<const uint32_t*>(lgs[x.lg].ptr);
        int idx = int(std::find(bin.begin(), bin.end(), p) - bin.begin());
        if (idx == int(bin.size())) bin.push_back(p);
        add(FOP_LOADB, reg_base, idx, 0);
        return reg_base;
      }
      case E_THRESH: {
        const uint16_t* p = static_cast<const uint16_t*>(lgs[x.lg].ptr);
        int idx = int(std::find(uin.begin(), uin.end(), p) - uin.begin());
        if (idx == int(uin.size())) uin.push_back(p);
        add(FOP_THRESH, reg_base, idx, 0, x.lo, x.hi);
        return reg_base;
      }
      case E_NOT: {
        int r = compile_expr(x.a, fp, bin, uin, reg_base);
        add(FOP_NOT, r, r, 0);
        return r;
      }
      default: {
        // Sethi-Ullman: evaluate the more demanding child first
        int first = x.a, second = x.b;
        if (exprs[x.b].need > exprs[x.a].need) std::swap(first, second);
        int r1 = compile_expr(first, fp, bin, uin, reg_base);
        int r2 = compile_expr(second, fp, bin, uin, reg_base + 1);
        add(x.k == E_AND ? FOP_AND : FOP_OR, r1, r1, r2);
        return r1;
      }
    }
  }

  int enqueue(cudaStream_t st) {
    int launches = 0;
    cudaMemsetAsync(d_err, 0, sizeof(int), st);
    size_t tl_n = 0;
    if (timeline) {
      tl_step.assign(lgs.size(), -1);
      cuda_check(cudaEventRecord(tl_event(tl_n++), st), "timeline");
    }
    struct TimelineMark {  // after every step (break/continue included)
      slcs_program* p;
      cudaStream_t st;
      size_t& n;
      int q;
      ~TimelineMark() {
        if (!p->timeline || q < 0) return;
        const LG& m = p->lgs[size_t(q)];
        const int lead = m.group >= 0 ? m.group : q;
        if (lead != q && p->tl_step[size_t(lead)] >= 0) {  // emitted with its group lead
          p->tl_step[size_t(q)] = p->tl_step[size_t(lead)];
          return;
        }
        cudaEventRecord(p->tl_event(n), st);
        p->tl_step[size_t(q)] = int(n) - 1;
        ++n;
      }
    };
    // `through` of the reach launched just before (null after any other step):
    // a reach on the same `through` may read it before its launch dependency
    const void* prev_through = nullptr;
    for (int qi : exec_order) {
      const size_t q = size_t(qi);
      LG& n = lgs[q];
      if (n.dead || n.kind == LG_INPUT) continue;
      TimelineMark tl_mark{this, st, tl_n, int(q)};
      const void* cur_through = n.kind == LG_REACH && n.in.size() > 1 ? lgs[n.in[1]].ptr : nullptr;
      const bool early_through = cur_through && cur_through == prev_through;
      prev_through = cur_through;
      bool bad = false;
      for (int i : n.in)
        if (!lgs[i].ptr) bad = true;
      if (bad) continue;
      Geo gb = bool_geo(n.w, n.h, n.batch);
      switch (n.kind) {
        case LG_EW: {
          if (n.group >= 0 && n.group != int(q)) break;  // emitted with its group lead
          std::vector<int> members = group_members(int(q), bad);
          if (bad) break;
          FusedProgram fp;
          std::vector<const uint32_t*> bin;
          std::vector<const uint16_t*> uin;
          fwd_.clear();
          int saved_reg = kFusedRegs;
          for (size_t i = 0; i < members.size(); ++i) {
            const LG& m = lgs[members[i]];
            const int r = compile_expr(m.expr, fp, bin, uin, 0);
            FusedOp st_op;
            st_op.op = FOP_STORE;
            st_op.dst = uint8_t(r);
            st_op.a = uint8_t(i);
            st_op.b = 0;
            st_op.lo = st_op.hi = 0;
            fp.ops[fp.n_ops++] = st_op;
            fp.out[i] = static_cast<uint32_t*>(m.ptr);
            for (size_t k = i + 1; k < members.size(); ++k)
              if (std::find(lgs[members[k]].in.begin(), lgs[members[k]].in.end(), members[i]) !=
                  lgs[members[k]].in.end()) {
                FusedOp cp;
                cp.op = FOP_OR;
                cp.dst = uint8_t(--saved_reg);
                cp.a = cp.b = uint8_t(r);
                cp.lo = cp.hi = 0;
                fp.ops[fp.n_ops++] = cp;
                fwd_[members[i]] = saved_reg;
                break;
              }
          }
          fwd_.clear();
          for (size_t z = 0; z < bin.size(); ++z) fp.bin[z] = bin[z];
          fp.n_bin = int(bin.size());
          for (size_t z = 0; z < uin.size(); ++z) fp.uin[z] = uin[z];
          launches += launch_fused(fp, gb, u16_geo(n.w, n.h, n.batch), st);
          break;
        }
        case LG_NEAR:
          launches += launch_near(static_cast<const uint32_t*>(lgs[n.in[0]].ptr),
                                  static_cast<uint32_t*>(n.ptr), gb, n.k, n.erode, st);
          break;
        case LG_THRESH_DEV:
          launches += launch_threshold_dev(static_cast<const uint16_t*>(lgs[n.in[0]].ptr),
                                           static_cast<uint32_t*>(n.ptr),
                                           u16_geo(n.w, n.h, n.batch), gb, n.cmp,
                                           d_nums + n.num_a, st);
          break;
        case LG_LABELS: {
          size_t lb = round_up(ccl_labels_bytes(n.w, n.h, n.batch), 256);
          cudaMemsetAsync(static_cast<char*>(n.ptr) + lb, 0, n.bytes - lb, st);
          launches += launch_labels(static_cast<const uint32_t*>(lgs[n.in[0]].ptr), n.ptr, gb, st);
          break;
        }
        case LG_REACH: {
          if (n.group >= 0) {  // a batch of independent small reaches
            if (n.group != int(q)) break;
            std::vector<int> members = group_members(int(q), bad);
            if (bad) break;
            const uint32_t* tg[4];
            const uint32_t* th[4];
            uint32_t* ou[4];
            for (size_t i = 0; i < members.size(); ++i) {
              const LG& m = lgs[members[i]];
              tg[i] = static_cast<const uint32_t*>(lgs[m.in[0]].ptr);
              th[i] = static_cast<const uint32_t*>(lgs[m.in[1]].ptr);
              ou[i] = static_cast<uint32_t*>(m.ptr);
            }
            launches += launch_reach_small_multi(tg, th, ou, int(members.size()), gb, st);
            break;
          }
          if (n.gen_idx >= 0 && n.chain_len > 1) {
            const LG& lab = lgs[n.in[2]];
            size_t lb = round_up(ccl_labels_bytes(n.w, n.h, n.batch), 256);
            launches += launch_reach_chain(
                static_cast<const uint32_t*>(lgs[n.in[0]].ptr),
                static_cast<const uint32_t*>(lgs[n.in[1]].ptr), lab.ptr,
                reinterpret_cast<uint32_t*>(static_cast<char*>(lab.ptr) + lb),
                uint32_t(n.chain_idx0), n.chain_len, n.chain_kmid, std::max(1, n.k),
                static_cast<uint32_t*>(n.ptr), static_cast<uint32_t*>(scratch), gb, st);
            break;
          }
          if (n.gen_idx >= 0) {
            const LG& lab = lgs[n.in[2]];
            size_t lb = round_up(ccl_labels_bytes(n.w, n.h, n.batch), 256);
            launches += launch_reach_labeled(
                static_cast<const uint32_t*>(lgs[n.in[0]].ptr),
                static_cast<const uint32_t*>(lgs[n.in[1]].ptr), lab.ptr,
                reinterpret_cast<uint32_t*>(static_cast<char*>(lab.ptr) + lb),
                uint32_t(n.gen_idx), static_cast<uint32_t*>(n.ptr),
                static_cast<uint32_t*>(scratch), gb, st, n.k);
            break;
          }
          CclScratch cs;
          ccl_scratch_carve(scratch, n.w, n.h, n.batch, true, false, &cs);
          size_t sb = ccl_scratch_bytes(n.w, n.h, n.batch, true, false);
          uint32_t* tmp = ccl_small_path(n.w, n.h)
                              ? nullptr
                              : reinterpret_cast<uint32_t*>(static_cast<char*>(scratch) + sb);
          launches += launch_reach(static_cast<const uint32_t*>(lgs[n.in[0]].ptr),
                                   static_cast<const uint32_t*>(lgs[n.in[1]].ptr),
                                   static_cast<uint32_t*>(n.ptr), tmp, gb, cs, st, n.k, n.tk,
                                   early_through);
          break;
        }
        case LG_CCL: {
          CclScratch cs;  // sizes hold the components' max keys
          ccl_scratch_carve(scratch, n.w, n.h, n.batch, false, true, &cs);
          launches += launch_ccl(static_cast<const uint32_t*>(lgs[n.in[0]].ptr),
                                 static_cast<uint32_t*>(n.ptr), gb, cs, st);
          break;
        }
        case LG_MAXVOL: {
          if (n.pro_expr >= 0 || n.epi_expr >= 0) {
            FusedProgram pro, epi;
            if (n.pro_expr >= 0) pro = listing(n.pro_expr, -1);
            if (n.epi_expr >= 0) epi = listing(n.epi_expr, n.epi_src);
            launches += launch_maxvol_small_listing(
                n.pro_expr >= 0 ? &pro : nullptr, n.epi_expr >= 0 ? &epi : nullptr,
                n.pro_expr >= 0 ? nullptr : static_cast<const uint32_t*>(lgs[n.in[0]].ptr),
                static_cast<uint32_t*>(n.ptr), gb, st);
            break;
          }
          CclScratch cs;
          ccl_scratch_carve(scratch, n.w, n.h, n.batch, false, true, &cs);
          launches += launch_maxvol(static_cast<const uint32_t*>(lgs[n.in[0]].ptr),
                                    static_cast<uint32_t*>(n.ptr), gb, cs, st);
          break;
        }
        case LG_VOLUME: {
          // d_counts: 2 zeroed u64 per number slot (the first: the volume accumulator)
          if (n.group >= 0) {  // adjacent volumes: one launch
            if (n.group != int(q)) break;
            std::vector<int> members = group_members(int(q), bad);
            if (bad) break;
            VolumeJobs jobs{};
            for (const int mq : members) {
              const LG& m = lgs[size_t(mq)];
              jobs.job[jobs.n++] = VolumeJob{static_cast<const uint32_t*>(lgs[m.in[0]].ptr),
                                             bool_geo(m.w, m.h, 1).slice,
                                             d_counts + 2 * m.num_out, nullptr,
                                             d_nums + m.num_out};
            }
            launches += launch_volume_multi(jobs, st);
            break;
          }
          launches += launch_volume(static_cast<const uint32_t*>(lgs[n.in[0]].ptr), nullptr,
                                    d_nums + n.num_out, d_counts + 2 * n.num_out, gb, st);
          break;
        }
        case LG_ARITH:
          pdl(k_arith, 1, 1, 0, st, d_nums, n.num_a, n.num_b, n.ca, n.cb, n.num_out, n.aop, d_err,
                                   n.k + 1);
          ++launches;
          break;
        default: break;
      }
    }
    return launches;
  }

  void ensure_staging(size_t bytes) {
    if (staging_bytes >= bytes) return;
    if (staging) cudaFree(staging);
    staging = nullptr;
    cuda_check(cudaMalloc(&staging, bytes), "program staging");
    staging_bytes = bytes;
  }

  void run(int flags) {
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    const int fusion = (flags & 2) ? 0 : 1;
    const bool label_cse = fusion && !(flags & 4);
    const bool chain = label_cse && !(flags & 8);
    timeline = (flags & 16) != 0;
    if (timeline) flags &= ~1;  // eager launches: events between the steps
    const int mode = fusion | (label_cse ? 2 : 0) | (chain ? 4 : 0);
    if (!planned || planned_fusion != mode) plan(fusion, label_cse, chain);
    planned_fusion = mode;
    // order after work already queued on the context stream
    cuda_check(cudaEventRecord(ev_in, ctx->stream), "event");
    cuda_check(cudaStreamWaitEvent(pstream, ev_in, 0), "wait");
    for (auto& kv : inputs) {
      InputSlot& s = kv.second;
      // images are immutable (shared_ptr<const ImageBuffer>, image.hpp:74) and the
      // slot holds a reference, so a still-bound image that was already copied in
      // has not changed: skip the copy
      if (s.bound && s.copied != s.bound) {
        cuda_check(cudaMemcpyAsync(s.data, s.bound->data, s.bytes, cudaMemcpyDeviceToDevice,
                                   pstream),
                   "bind copy");
        s.copied = s.bound;
      }
    }
    int launches = 0;
    if (flags & 1) {
      if (!exec) {
        cuda_check(cudaStreamBeginCapture(pstream, cudaStreamCaptureModeThreadLocal), "capture");
        int n = 0;
        try {
          n = enqueue(pstream);
        } catch (...) {
          cudaGraph_t g;
          cudaStreamEndCapture(pstream, &g);
          if (g) cudaGraphDestroy(g);
          throw;
        }
        cuda_check(cudaStreamEndCapture(pstream, &graph), "end capture");
        cuda_check(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
        launches_per_run = n;
      }
      cuda_check(cudaGraphLaunch(exec, pstream), "graph launch");
      launches = launches_per_run;
    } else {
      launches = enqueue(pstream);
      launches_per_run = launches;
    }
    ctx->launches += launches;
    cuda_check(cudaEventRecord(ev_out, pstream), "event");
    cuda_check(cudaStreamWaitEvent(ctx->stream, ev_out, 0), "wait");
    cuda_check(cudaGetLastError(), "program launch");
    if (has_dev_arith) {
      int err = 0;
      cuda_check(cudaMemcpyAsync(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost, pstream), "err");
      cuda_check(cudaStreamSynchronize(pstream), "sync");
      if (err) {
        vals[err - 1].err = "division by zero";
        fail(SLCS_ERR_RUN, "task " + std::to_string(err - 1) + " (" + tasks[err - 1].opcode +
                               ") failed: division by zero");
      }
    }
    if (timeline && !tl_ev.empty()) {
      size_t used = 1;
      for (int v : tl_step) used = std::max(used, size_t(v + 2));
      cuda_check(cudaEventSynchronize(tl_ev[used - 1]), "timeline");
      tl_ms.assign(2 * (used - 1), 0.f);
      for (size_t i = 0; i + 1 < used; ++i) {
        cudaEventElapsedTime(&tl_ms[2 * i], tl_ev[0], tl_ev[i]);
        cudaEventElapsedTime(&tl_ms[2 * i + 1], tl_ev[0], tl_ev[i + 1]);
      }
    }
    if (first_fail >= 0) fail(SLCS_ERR_RUN, fail_msg);
  }

  const Val& result_val(int task) {
    if (!planned) fail(SLCS_ERR_RUN, "program has not run");
    if (task < 0 || task >= int(tasks.size())) fail(SLCS_ERR_ARG, "task id out of range");
    const Val& v = vals[task];
    if (!v.err.empty()) fail(SLCS_ERR_RUN, "task " + std::to_string(task) + " has no value: " + v.err);
    if (v.type != VT_NUM && (v.lg < 0 || !lgs[v.lg].ptr))
      fail(SLCS_ERR_ARG, "task " + std::to_string(task) +
                             " is not materialised (only save/print results are kept)");
    return v;
  }

  double number(const Val& v) {
    if (v.host_num) return v.num;
    double out = 0;
    cuda_check(cudaMemcpyAsync(&out, d_nums + v.numslot, sizeof(double), cudaMemcpyDeviceToHost,
                               pstream),
               "number readback");
    cuda_check(cudaStreamSynchronize(pstream), "sync");
    return out;
  }
};

// ============================================================================
extern "C" {

int slcs_program_create(slcs_ctx* ctx, int n_tasks, const char* const* opcodes,
                        const double* payload_num, const char* const* payload_str,
                        const int* dep_off, const int* deps, slcs_program** out) {
  return pguard([&] {
    if (!ctx || !out || n_tasks < 0 || (n_tasks && (!opcodes || !dep_off)))
      fail(SLCS_ERR_ARG, "invalid program arguments");
    auto* p = new slcs_program;
    try {
      p->ctx = ctx;
      for (int i = 0; i < n_tasks; ++i) {
        PTask t;
        t.opcode = opcodes[i] ? opcodes[i] : "";
        if (!parse_opcode(t.opcode, t.op, t.sub))
          fail(SLCS_ERR_RUN, "task " + std::to_string(i) + " (" + t.opcode +
                                 ") failed: unknown opcode '" + t.opcode + "'");
        if (payload_num) t.num = payload_num[i];
        if (payload_str && payload_str[i]) t.str = payload_str[i];
        for (int d = dep_off[i]; d < dep_off[i + 1]; ++d) {
          if (deps[d] < 0 || deps[d] >= i)
            fail(SLCS_ERR_ARG, "task " + std::to_string(i) + ": dependencies must have smaller ids");
          t.deps.push_back(deps[d]);
        }
        if (int(t.deps.size()) != op_arity(t.op))
          fail(SLCS_ERR_ARG, "task " + std::to_string(i) + " (" + t.opcode + "): wrong arity");
        if (t.op == OP_LOAD) p->inputs[t.str];
        p->tasks.push_back(std::move(t));
      }
      cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
      cuda_check(cudaStreamCreateWithFlags(&p->pstream, cudaStreamNonBlocking), "stream");
      cuda_check(cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming), "event");
      cuda_check(cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming), "event");
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

int slcs_program_destroy(slcs_program* prog) {
  return pguard([&] {
    if (!prog) return;
    cudaSetDevice(prog->ctx->device);
    cudaStreamSynchronize(prog->pstream);
    for (auto& kv : prog->inputs) {
      if (kv.second.data) cudaFree(kv.second.data);
      if (kv.second.bound) drop_image(const_cast<slcs_image*>(kv.second.bound));
    }
    prog->release_plan();
    if (prog->staging) cudaFree(prog->staging);
    cudaEventDestroy(prog->ev_in);
    cudaEventDestroy(prog->ev_out);
    cudaStreamDestroy(prog->pstream);
    delete prog;
  });
}

static InputSlot& input_slot(slcs_program* prog, const char* name, int kind, int w, int h,
                             int batch) {
  auto it = prog->inputs.find(name ? name : "");
  if (it == prog->inputs.end())
    fail(SLCS_ERR_ARG, std::string("no load task reads '") + (name ? name : "") + "'");
  InputSlot& s = it->second;
  if (s.kind != kind || s.w != w || s.h != h || s.batch != batch) {
    if (w < 1 || h < 1 || batch < 1) fail(SLCS_ERR_SHAPE, "bad input dimensions");
    cudaStreamSynchronize(prog->pstream);
    if (s.data) cudaFree(s.data);
    s.kind = kind;
    s.w = w;
    s.h = h;
    s.batch = batch;
    s.geo = kind == SLCS_U16 ? u16_geo(w, h, batch)
                             : (kind == SLCS_LABEL ? label_geo(w, h, batch) : bool_geo(w, h, batch));
    s.bytes = s.geo.slice * size_t(batch) * (kind == SLCS_U16 ? 2 : 4);
    cuda_check(cudaMalloc(&s.data, s.bytes), "program input slot");
    prog->planned = false;
    prog->release_plan();
  }
  return s;
}

int slcs_program_bind(slcs_program* prog, const char* name, const slcs_image* img) {
  return pguard([&] {
    if (!prog || !img) fail(SLCS_ERR_ARG, "null argument");
    std::lock_guard<std::mutex> lock(prog->mu);
    cuda_check(cudaSetDevice(prog->ctx->device), "cudaSetDevice");
    InputSlot& s = input_slot(prog, name, img->kind, img->geo.w, img->geo.h, img->geo.batch);
    const_cast<slcs_image*>(img)->refs.fetch_add(1);
    if (s.bound) drop_image(const_cast<slcs_image*>(s.bound));
    s.bound = img;
    s.copied = nullptr;
  });
}

int slcs_program_set_input_host(slcs_program* prog, const char* name, slcs_kind kind, int w,
                                int h, int batch, const void* host) {
  return pguard([&] {
    if (!prog || !host) fail(SLCS_ERR_ARG, "null argument");
    std::lock_guard<std::mutex> lock(prog->mu);
    cuda_check(cudaSetDevice(prog->ctx->device), "cudaSetDevice");
    InputSlot& s = input_slot(prog, name, kind, w, h, batch);
    if (s.bound) {
      drop_image(const_cast<slcs_image*>(s.bound));
      s.bound = nullptr;
    }
    s.copied = nullptr;
    cudaStream_t st = prog->pstream;
    if (kind == SLCS_U16) {
      // one dense H2D copy (many short pitched rows are slow over PCIe), then
      // a device-side repitch
      const size_t dense = size_t(w) * size_t(h) * size_t(batch) * 2;
      if (s.geo.pitch == size_t(w)) {
        cuda_check(cudaMemcpyAsync(s.data, host, dense, cudaMemcpyHostToDevice, st),
                   "input upload");
      } else {
        prog->ensure_staging(dense);
        cuda_check(cudaMemcpyAsync(prog->staging, host, dense, cudaMemcpyHostToDevice, st),
                   "input upload");
        prog->ctx->launches += launch_repitch_u16(
            static_cast<const uint16_t*>(prog->staging), size_t(w), static_cast<uint16_t*>(s.data),
            s.geo.pitch, w, size_t(h) * size_t(batch), st);
      }
    } else if (kind == SLCS_LABEL) {
      cuda_check(cudaMemcpyAsync(s.data, host, size_t(w) * h * batch * 4, cudaMemcpyHostToDevice,
                                 st),
                 "input upload");
    } else {
      size_t npx = size_t(w) * size_t(h) * size_t(batch);
      prog->ensure_staging(npx);
      cuda_check(cudaMemcpyAsync(prog->staging, host, npx, cudaMemcpyHostToDevice, st),
                 "input upload");
      prog->ctx->launches += launch_pack_u8(static_cast<const uint8_t*>(prog->staging),
                                            static_cast<uint32_t*>(s.data), s.geo, true, st);
    }
  });
}

int slcs_program_run(slcs_program* prog, int flags) {
  return pguard([&] {
    if (!prog) fail(SLCS_ERR_ARG, "null program");
    std::lock_guard<std::mutex> lock(prog->mu);
    prog->run(flags);
  });
}

int slcs_program_download(slcs_program* prog, int task, void* host, size_t bytes) {
  return pguard([&] {
    if (!prog || !host) fail(SLCS_ERR_ARG, "null argument");
    std::lock_guard<std::mutex> lock(prog->mu);
    cuda_check(cudaSetDevice(prog->ctx->device), "cudaSetDevice");
    const Val& v = prog->result_val(task);
    if (v.type == VT_NUM) {
      if (bytes < sizeof(double)) fail(SLCS_ERR_ARG, "buffer too small");
      double d = prog->number(v);
      std::memcpy(host, &d, sizeof(double));
      return;
    }
    const LG& n = prog->lgs[v.lg];
    size_t npx = size_t(n.w) * size_t(n.h) * size_t(n.batch);
    cudaStream_t st = prog->pstream;
    if (v.type == VT_BOOL) {
      if (bytes < npx) fail(SLCS_ERR_ARG, "buffer too small");
      prog->ensure_staging(npx);
      Geo g = bool_geo(n.w, n.h, n.batch);
      prog->ctx->launches += launch_unpack(static_cast<const uint32_t*>(n.ptr),
                                           static_cast<uint8_t*>(prog->staging), g, st);
      cuda_check(cudaMemcpyAsync(host, prog->staging, npx, cudaMemcpyDeviceToHost, st), "d2h");
    } else if (v.type == VT_U16) {
      if (bytes < npx * 2) fail(SLCS_ERR_ARG, "buffer too small");
      Geo g = u16_geo(n.w, n.h, n.batch);
      const void* src = n.ptr;
      if (g.pitch != size_t(n.w)) {  // dense on the device first: one D2H copy
        prog->ensure_staging(npx * 2);
        prog->ctx->launches += launch_repitch_u16(static_cast<const uint16_t*>(n.ptr), g.pitch,
                                                  static_cast<uint16_t*>(prog->staging),
                                                  size_t(n.w), n.w, size_t(n.h) * n.batch, st);
        src = prog->staging;
      }
      cuda_check(cudaMemcpyAsync(host, src, npx * 2, cudaMemcpyDeviceToHost, st), "d2h");
    } else {
      if (bytes < npx * 4) fail(SLCS_ERR_ARG, "buffer too small");
      cuda_check(cudaMemcpyAsync(host, n.ptr, npx * 4, cudaMemcpyDeviceToHost, st), "d2h");
    }
    cuda_check(cudaStreamSynchronize(st), "sync");
  });
}

int slcs_program_result(slcs_program* prog, int task, int* kind_out, slcs_image** img_out,
                        double* num_out) {
  return pguard([&] {
    if (!prog) fail(SLCS_ERR_ARG, "null program");
    std::lock_guard<std::mutex> lock(prog->mu);
    cuda_check(cudaSetDevice(prog->ctx->device), "cudaSetDevice");
    const Val& v = prog->result_val(task);
    if (v.type == VT_NUM) {
      if (kind_out) *kind_out = 1;
      if (num_out) *num_out = prog->number(v);
      if (img_out) *img_out = nullptr;
      return;
    }
    if (kind_out) *kind_out = 0;
    if (!img_out) return;
    const LG& n = prog->lgs[v.lg];
    int kind = v.type == VT_U16 ? SLCS_U16 : (v.type == VT_LABEL ? SLCS_LABEL : SLCS_BOOL);
    slcs_image* img = new_image(prog->ctx, kind, n.w, n.h, n.batch);
    // the image is allocated on the context stream; copy after the program
    cuda_check(cudaEventRecord(prog->ev_out, prog->pstream), "event");
    cuda_check(cudaStreamWaitEvent(prog->ctx->stream, prog->ev_out, 0), "wait");
    cuda_check(cudaMemcpyAsync(img->data, n.ptr, img->bytes, cudaMemcpyDeviceToDevice,
                               prog->ctx->stream),
               "result copy");
    *img_out = img;
  });
}

int slcs_program_task_state(slcs_program* prog, int task, int* state, const char** message) {
  return pguard([&] {
    if (!prog || !state) fail(SLCS_ERR_ARG, "null argument");
    std::lock_guard<std::mutex> lock(prog->mu);
    if (!prog->planned) fail(SLCS_ERR_RUN, "program has not run");
    if (task < 0 || task >= int(prog->tasks.size())) fail(SLCS_ERR_ARG, "task id out of range");
    const Val& v = prog->vals[task];
    *state = v.err.empty() ? 0 : (v.aborted ? 2 : 1);
    if (message) *message = v.err.c_str();
  });
}

int slcs_program_task_time(slcs_program* prog, int task, float* start_ms, float* end_ms) {
  return pguard([&] {
    if (!prog || !start_ms || !end_ms) fail(SLCS_ERR_ARG, "null argument");
    std::lock_guard<std::mutex> lock(prog->mu);
    if (task < 0 || task >= int(prog->tasks.size())) fail(SLCS_ERR_ARG, "task id out of range");
    *start_ms = *end_ms = -1.f;
    if (!prog->timeline || prog->vals.size() != prog->tasks.size()) return;
    const int lg = prog->vals[task].lg;
    if (lg < 0 || size_t(lg) >= prog->tl_step.size()) return;
    const int st = prog->tl_step[size_t(lg)];
    if (st < 0 || size_t(2 * st + 1) >= prog->tl_ms.size()) return;
    *start_ms = prog->tl_ms[size_t(2 * st)];
    *end_ms = prog->tl_ms[size_t(2 * st + 1)];
  });
}

int slcs_program_launches(slcs_program* prog, int* out) {
  return pguard([&] {
    if (!prog || !out) fail(SLCS_ERR_ARG, "null argument");
    *out = prog->launches_per_run;
  });
}

const char* slcs_program_plan(slcs_program* prog) {
  return prog ? prog->plan_text.c_str() : "";
}

}  // extern "C"
