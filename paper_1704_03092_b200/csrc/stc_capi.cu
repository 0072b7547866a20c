// stc_capi.cu -- the C ABI (include/stc_b200.h): host-side planning of the
// Strassen contraction and the kernel launch sequence for each variant.
//
// Planning mirrors strassen.contract (strassen.py:141-207):
//   views of A (I x P), B (P x J), C (I x J)          strassen.py:156-161
//   quadrants with PAD padding to 2^L                   strassen.py:101-127
//   7^L terms by level-1 substitution                   strassen.py:70-94
// and replaces the CPU cache-blocking (driver.py:76-126) with one persistent
// DMMA launch over all (term, tile) work items (ABC) or batched launches that
// write dense M slots (AB / Naive).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "stc_internal.cuh"

using namespace stc;

extern "C" char **environ;

namespace {

// getenv for the STC_* knobs, memoised per thread: the planner and the per-call path
// consult ~20 of them per call, and a getenv scans the whole environment.  The memo is
// dropped whenever the environment array changes (a putenv / setenv -- Python's
// os.environ -- replaces an entry pointer; env_refresh compares the pointer array).
struct EnvMemo {
  std::vector<char *> snap;
  std::vector<std::pair<const char *, const char *>> vals;  // (knob name literal, value)
};
thread_local EnvMemo g_env;

void env_refresh() {
  size_t n = 0;
  while (environ && environ[n]) ++n;
  if (n == g_env.snap.size() && std::equal(g_env.snap.begin(), g_env.snap.end(), environ)) return;
  g_env.snap.assign(environ, environ + n);
  g_env.vals.clear();
}

const char *stc_env(const char *name) {
  for (const auto &kv : g_env.vals)
    if (kv.first == name || strcmp(kv.first, name) == 0) return kv.second;
  const char *v = getenv(name);
  g_env.vals.emplace_back(name, v);
  return v;
}

thread_local std::string g_err;
thread_local cudaEvent_t g_ev_before = nullptr, g_ev_after = nullptr;  // stc_set_kernel_events
thread_local const int32_t *g_c_ready = nullptr;                        // stc_set_c_ready
thread_local stc::SlotOverride g_slot_ovr;                                // stc::set_slot_override
thread_local bool g_slot_ovr_set = false;

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char *what) {
  return fail(STC_ECUDA, "CUDA error in %s: %s", what, cudaGetErrorString(e));
}

#define CU(expr, what)                       \
  do {                                       \
    cudaError_t _e = (expr);                 \
    if (_e != cudaSuccess) return cuda_fail(_e, what); \
  } while (0)

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
int64_t rup(int64_t a, int64_t b) { return cdiv(a, b) * b; }
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

int64_t bundle_len(const stc_bundle &b) {
  int64_t n = 1;
  for (int d = 0; d < b.nlab; ++d) n *= b.ext[d];
  return n;
}

// ---------------------------------------------------------------- staging
// Pinned host staging for the small plan tables, double-buffered and fenced
// by events so uploads never force a stream synchronisation.
// Page-locked staging ring for the plan tables.  A slot is reused once the
// k_stage launch that read it has run; when every slot is still pending (a
// stream parked behind transfers, as in stc_contract_host) the ring grows
// instead of blocking the host, up to kStagingMax slots.
constexpr int kStagingMax = 64;
struct Staging {
  void *host[kStagingMax] = {};
  size_t cap[kStagingMax] = {};
  cudaEvent_t ev[kStagingMax] = {};
  bool used[kStagingMax] = {};
  int nslots = 0, next = 0;
  std::mutex mu;
};
Staging g_staging[64];
thread_local int64_t g_stage_launches = 0;  // k_stage launches of the current call

// Host table -> device, read by a k_stage launch from a staging slot;
// optionally zeroes [zero, zero + zero_bytes) in the same launch.
int upload(const void *src, size_t bytes, void *dst, cudaStream_t s, void *zero = nullptr, size_t zero_bytes = 0) {
  if (bytes == 0 && zero_bytes == 0) return STC_OK;
  int dev = 0;
  CU(cudaGetDevice(&dev), "cudaGetDevice");
  Staging &st = g_staging[dev & 63];
  std::lock_guard<std::mutex> lk(st.mu);
  int i = -1;
  for (int t = 0; t < st.nslots && i < 0; ++t) {  // a free slot, oldest first
    const int c = (st.next + t) % st.nslots;
    if (!st.used[c] || cudaEventQuery(st.ev[c]) == cudaSuccess) i = c;
  }
  cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not an error here
  if (i < 0 && st.nslots < kStagingMax) i = st.nslots++;
  if (i < 0) {  // ring full: wait for the oldest
    i = st.next % st.nslots;
    CU(cudaEventSynchronize(st.ev[i]), "cudaEventSynchronize");
  }
  st.next = (i + 1) % std::max(st.nslots, 1);
  if (!st.ev[i]) CU(cudaEventCreateWithFlags(&st.ev[i], cudaEventDisableTiming), "cudaEventCreate");
  if (st.cap[i] < bytes) {
    if (st.used[i]) CU(cudaEventSynchronize(st.ev[i]), "cudaEventSynchronize");
    if (st.host[i]) cudaFreeHost(st.host[i]);
    st.host[i] = nullptr;
    size_t c = std::max<size_t>(bytes, 1 << 16);
    CU(cudaMallocHost(&st.host[i], c), "cudaMallocHost");
    st.cap[i] = c;
  }
  if (bytes) memcpy(st.host[i], src, bytes);
  CU(launch_stage(st.host[i], dst, bytes, zero, zero_bytes, s), "k_stage");
  ++g_stage_launches;
  CU(cudaEventRecord(st.ev[i], s), "cudaEventRecord");
  st.used[i] = true;
  return STC_OK;
}

// ------------------------------------------------------------ Strassen terms
struct Op {
  int q, s;
};
struct Term {
  std::vector<Op> a, b, c;
};

// strassen.py:56-65
const int kL1[7][3][2][2] = {
    {{{0, 1}, {3, 1}}, {{0, 1}, {3, 1}}, {{0, 1}, {3, 1}}},
    {{{2, 1}, {3, 1}}, {{0, 1}, {0, 0}}, {{2, 1}, {3, -1}}},
    {{{0, 1}, {0, 0}}, {{1, 1}, {3, -1}}, {{1, 1}, {3, 1}}},
    {{{3, 1}, {0, 0}}, {{2, 1}, {0, -1}}, {{0, 1}, {2, 1}}},
    {{{0, 1}, {1, 1}}, {{3, 1}, {0, 0}}, {{1, 1}, {0, -1}}},
    {{{2, 1}, {0, -1}}, {{0, 1}, {1, 1}}, {{3, 1}, {0, 0}}},
    {{{1, 1}, {3, -1}}, {{2, 1}, {3, 1}}, {{0, 1}, {0, 0}}},
};

// strassen.py:70-94: level l = level-1 table (outer) x level l-1 table (inner),
// quadrant q*4^(l-1) + q2, sign s*s2.
std::vector<Term> strassen_terms(int level) {
  std::vector<Term> terms(1);
  terms[0].a = {{0, 1}};
  terms[0].b = {{0, 1}};
  terms[0].c = {{0, 1}};
  for (int lev = 1; lev <= level; ++lev) {
    int mult = 1;
    for (int i = 1; i < lev; ++i) mult *= 4;
    std::vector<Term> next;
    next.reserve(terms.size() * 7);
    for (int o = 0; o < 7; ++o)
      for (const Term &in : terms) {
        Term t;
        for (int side = 0; side < 3; ++side) {
          const std::vector<Op> &inner = side == 0 ? in.a : side == 1 ? in.b : in.c;
          std::vector<Op> &dst = side == 0 ? t.a : side == 1 ? t.b : t.c;
          for (int e = 0; e < 2; ++e) {
            if (kL1[o][side][e][1] == 0) continue;
            for (const Op &x : inner) dst.push_back({kL1[o][side][e][0] * mult + x.q, kL1[o][side][e][1] * x.s});
          }
        }
        next.push_back(std::move(t));
      }
    terms.swap(next);
  }
  return terms;
}

// quadrant id (row-major per level, top level most significant) -> (row, col)
void quad_rc(int q, int level, int64_t &r, int64_t &c) {
  r = 0;
  c = 0;
  for (int l = 0; l < level; ++l) {
    const int d = (q >> (2 * (level - 1 - l))) & 3;
    r = r * 2 + (d >> 1);
    c = c * 2 + (d & 1);
  }
}

// ---------------------------------------------------------- tile ordering
// Quadrant-local box of a bundle and the tile order of its dims (DESIGN.md
// "tile ordering").  The permutation is applied identically to every quadrant
// and to both tensors sharing the bundle, so quadrants and their pairing are
// exactly the reference's; only the grouping of indices into GPU tiles moves.
struct Tiling {
  int nbox = 0;
  int64_t box_ext[STC_MAX_LABELS];
  int32_t order[STC_MAX_LABELS];
};

Tiling make_tiling(const stc_bundle &b, int level, const int64_t *key, bool reference) {
  Tiling t;
  if (reference) return t;
  const int64_t n = bundle_len(b);
  const int64_t Q = (int64_t)1 << level;
  if (n % Q != 0) return t;  // padded quadrants: keep the reference order
  const int64_t xq = n / Q;
  int64_t P = 1;
  int k = 0;
  while (k < b.nlab && xq % (P * b.ext[k]) == 0) P *= b.ext[k++];
  const int64_t c = xq / P;
  if (k < b.nlab && b.ext[k] % c != 0) return t;
  if (k == b.nlab && c != 1) return t;
  int64_t ext[STC_MAX_LABELS + 1], ks[STC_MAX_LABELS + 1];
  int nd = 0;
  for (int d = 0; d < k; ++d) {
    ext[nd] = b.ext[d];
    ks[nd++] = key[d] < 0 ? -key[d] : key[d];
  }
  if (c > 1) {
    ext[nd] = c;
    ks[nd++] = key[k] < 0 ? -key[k] : key[k];
  }
  if (nd > STC_MAX_LABELS) return t;
  std::vector<int> idx(nd);
  for (int i = 0; i < nd; ++i) idx[i] = i;
  std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return ks[x] < ks[y]; });
  t.nbox = nd;
  for (int i = 0; i < nd; ++i) {
    t.box_ext[i] = ext[i];
    t.order[i] = idx[i];
  }
  return t;
}

// Which bundle holds a tensor's smallest stride (extent > 1 labels only):
// returns 0 for the row bundle, 1 for the column bundle, -1 if none.
int min_stride_side(const stc_bundle &r, const stc_bundle &c) {
  int64_t best = INT64_MAX;
  int side = -1;
  for (int s = 0; s < 2; ++s) {
    const stc_bundle &b = s == 0 ? r : c;
    for (int d = 0; d < b.nlab; ++d) {
      if (b.ext[d] <= 1) continue;
      const int64_t v = b.str[d] < 0 ? -b.str[d] : b.str[d];
      if (v < best) {
        best = v;
        side = s;
      }
    }
  }
  return side;
}

VecDesc vec_bundle(const stc_bundle &b, int64_t base, int64_t nq, int64_t tile, const Tiling &t) {
  VecDesc d;
  memset(&d, 0, sizeof(d));
  d.mode = 0;
  d.len = bundle_len(b);
  d.nq = nq;
  d.q_len = cdiv(d.len, nq);  // pad_view to a multiple of 2^L, then split
  d.q_len_pad = rup(d.q_len, tile);
  d.base = base;
  d.nlab = b.nlab;
  for (int i = 0; i < b.nlab; ++i) {
    d.ext[i] = b.ext[i];
    d.str[i] = b.str[i];
  }
  d.nbox = t.nbox;
  for (int i = 0; i < t.nbox; ++i) {
    d.box_ext[i] = t.box_ext[i];
    d.order[i] = t.order[i];
  }
  return d;
}

// Per-slot x vectors (mode 2, slot stride = the slot size): a term's op addresses
// its own slot block of packed operand sums through the pool alone.
VecDesc slot_vec(int64_t len, int64_t stride, int64_t slot, int64_t nslots) {
  VecDesc d;
  memset(&d, 0, sizeof(d));
  d.mode = 2;
  d.nq = nslots;
  d.q_len = d.q_len_pad = d.len = len;
  d.stride = stride;
  d.base = slot;
  return d;
}

VecDesc vec_affine(int64_t len, int64_t len_pad, int64_t stride) {
  VecDesc d;
  memset(&d, 0, sizeof(d));
  d.mode = 1;
  d.nq = 1;
  d.q_len = len;
  d.q_len_pad = len_pad;
  d.len = len;
  d.stride = stride;
  return d;
}

int check_bundle(const stc_bundle &b, const char *name) {
  if (b.nlab < 0 || b.nlab > STC_MAX_LABELS) return fail(STC_EINVAL, "bundle %s: label count %d out of range", name, b.nlab);
  for (int d = 0; d < b.nlab; ++d)
    if (b.ext[d] < 1) return fail(STC_EINVAL, "bundle %s: extents must be positive", name);
  return STC_OK;
}

bool same_extents(const stc_bundle &x, const stc_bundle &y) {
  if (x.nlab != y.nlab) return false;
  for (int d = 0; d < x.nlab; ++d)
    if (x.ext[d] != y.ext[d]) return false;
  return true;
}

// Fast-index step of a gather pass's source (stc_internal.cuh FastMap): for a bundle
// kept in the reference order (first label fastest) whose unit-stride label u is not
// its first, the quadrant-local step that advances u by one (the product of the
// extents before it); 0 otherwise.  `group`: the t values per run, a power of two
// up to 4 (a 32-byte sector) and up to the extent of u and the runs a quadrant holds.
int64_t unit_step(const stc_bundle &b, const Tiling &t, int64_t fast_len, int &group) {
  group = 0;
  if (t.nbox > 0) return 0;  // tile order: the unit-stride label already leads
  int64_t mult = 1;
  for (int d = 0; d < b.nlab; ++d) {
    const int64_t s = b.str[d] < 0 ? -b.str[d] : b.str[d];
    if (s == 1 && b.ext[d] > 1) {
      if (d == 0 || mult < 8) return 0;
      const int64_t runs = std::min<int64_t>(b.ext[d], cdiv(fast_len, mult));
      int g = 1;
      while (g < 4 && 2 * g <= runs) g *= 2;
      if (g < 2) return 0;
      group = g;
      return mult;
    }
    mult *= b.ext[d];
  }
  return 0;
}

// ---------------------------------------------------------------- the plan
// Device snapshots of a plan's constant workspace region (scatter vectors, chunk
// strides, map coordinates, tables, accumulate lists, zeroed tickets and counters),
// one per operand mode (own views / repacked).  The first call of a plan builds the
// region in its workspace and copies it here; later calls restore it with one kernel
// (k_restore) instead of the 5-10 small launches that build it.  Shared by the copies
// of a cached plan; freed with the last one.
//
// Small problems also keep executable CUDA graphs of their launch sequence (restore,
// operand sums, DMMA kernel, accumulate), keyed by the operand / workspace pointers:
// a repeated call replays one graph instead of re-deriving and issuing 4+ launches
// (the host work would otherwise exceed the device time of a 576^3 contraction).
struct GraphKey {
  const void *a, *b, *c, *ws;
  int dev;
  int mode;  // the operand mode the pointers imply (its snapshot orders the replays)
  bool operator==(const GraphKey &o) const {
    return a == o.a && b == o.b && c == o.c && ws == o.ws && dev == o.dev;
  }
};
struct Resident {
  std::mutex mu;
  void *buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int dev[2] = {-1, -1};
  static constexpr size_t kGraphs = 8;
  struct Graph {
    GraphKey key;
    cudaGraphExec_t exec;
    stc_stats st;
  };
  std::vector<Graph> graphs;
  size_t graph_next = 0;
  ~Resident() {
    // cudaFree waits for the device's pending work (the graphs' replays read buf)
    for (int i = 0; i < 2; ++i) {
      if (buf[i]) cudaFree(buf[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
    }
    for (Graph &g : graphs) cudaGraphExecDestroy(g.exec);
  }
  // Launch the graph of `key` on s; false if there is none (or the launch failed).
  bool replay(const GraphKey &key, cudaStream_t s, stc_stats &st) {
    std::lock_guard<std::mutex> lk(mu);
    for (const Graph &g : graphs)
      if (g.key == key) {
        if (!order(g.key.mode, s) || cudaGraphLaunch(g.exec, s) != cudaSuccess) {
          cudaGetLastError();
          return false;
        }
        st = g.st;
        return true;
      }
    return false;
  }
  void keep(const GraphKey &key, cudaGraphExec_t exec, const stc_stats &st) {
    std::lock_guard<std::mutex> lk(mu);
    if (graphs.size() < kGraphs) {
      graphs.push_back({key, exec, st});
      return;
    }
    cudaGraphExecDestroy(graphs[graph_next].exec);  // freed once its pending launches ran
    graphs[graph_next] = {key, exec, st};
    graph_next = (graph_next + 1) % kGraphs;
  }
  // The snapshot of `mode` on device d, ordered before the work next enqueued on s; null if none.
  const void *ready(int mode, int d, cudaStream_t s) {
    if (stc_env("STC_NO_SNAPSHOT")) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    if (!buf[mode] || dev[mode] != d) return nullptr;
    if (!order(mode, s)) return nullptr;
    return buf[mode];
  }
  // s ordered after the snapshot copy of `mode` (a stream wait until the copy is known
  // complete; none after that).  Caller holds mu.
  bool order(int mode, cudaStream_t s) {
    if (settled[mode]) return true;
    if (cudaEventQuery(ev[mode]) == cudaSuccess) {
      settled[mode] = true;
      return true;
    }
    cudaGetLastError();  // (cudaErrorNotReady)
    if (cudaStreamWaitEvent(s, ev[mode], 0) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return true;
  }
  bool settled[2] = {false, false};
  // Copy [ws, ws + bytes) (complete in stream order on s) into a new snapshot of `mode`.
  cudaError_t save(int mode, int d, const void *ws, size_t bytes, cudaStream_t s) {
    if (stc_env("STC_NO_SNAPSHOT")) return cudaSuccess;
    std::lock_guard<std::mutex> lk(mu);
    if (buf[mode] || bytes == 0) return cudaSuccess;
    void *p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {  // no snapshot: later calls rebuild
      cudaGetLastError();
      return cudaSuccess;
    }
    cudaEvent_t e = nullptr;
    cudaError_t r = launch_restore(ws, p, bytes, s);
    if (r == cudaSuccess) r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (r == cudaSuccess) r = cudaEventRecord(e, s);
    if (r != cudaSuccess) {
      cudaFree(p);
      if (e) cudaEventDestroy(e);
      return r;
    }
    buf[mode] = p;
    ev[mode] = e;
    dev[mode] = d;
    return cudaSuccess;
  }
};

struct Plan {
  int level = 0, variant = 0;
  uint32_t flags = 0;
  int64_t m = 0, n = 0, k = 0;
  int64_t mq = 0, nq = 0, kq = 0, mq_pad = 0, nq_pad = 0, kq_pad = 0;
  int64_t Q = 1;  // quadrants per dimension
  int nquads = 1;
  int a_kfast = 0, b_kfast = 0;
  int64_t a_ustep = 0, b_ustep = 0;  // gather passes: fast-index step of the unit-stride label (FastMap)
  int a_ugroup = 0, b_ugroup = 0;
  Tiling ti, tj, tp;  // tile orders of the I, J, P bundles
  std::vector<VecDesc> vecs;
  int64_t pool_len = 0;
  int64_t ar = 0, ac = 0, br = 0, bc = 0, cr = 0, cc = 0;  // pool starts
  int64_t dxa = 0, dka = 0, dxb = 0, dkb = 0;              // Naive packed-operand vectors
  std::vector<Term> terms;
  // execution tables
  std::vector<TermDesc> tdesc;  // ABC: exec order; AB/Naive: per batch-local slot (rebuilt per batch)
  std::vector<OpDesc> ops;
  std::vector<TgtDesc> tgts;
  int batch = 1, nbatches = 1;
  int grid = 1;
  // workspace layout (bytes)
  int max_ops = 1;  // most views on one side of any term (2^L)
  size_t off_kbs = 0, off_coords = 0, off_mscr = 0, off_pka = 0, off_pkb = 0;
  bool need_pack = false;  // fused kernel on repacked operands (layout not box-regular)
  int stage_cap = 0;       // stc_problem.tiling: cap on the fused ring depth (0: none)
  int tshape = 0;          // fused kernel CTA tile shape (stc_fused.cu Shape): 0 128 x 128, 1 64 x 256, 2 256 x 64, 3 64 x 128, 4 128 x 64
  int64_t tm = BM, tn = BN;  // its tile rows / columns (quadrants padded to them)
  // ABC with C updated straight from the kernel, ticket-ordered per C tile; false for AB,
  // Naive and the dense-M ABC mode (many terms in flight per tile: dense M slots, then one
  // ordered accumulate pass -- the same additions in the same order, without ticket chains)
  bool ticketed = false;
  // ABC with pre-summed operands (k_presum): the 7^L operand sums of each side are
  // formed once per element position into per-term slots (term batches under the
  // workspace cap), and the fused kernel runs every term with one view per side
  bool presum = false;
  // which sides come from slots (bit 0 A, bit 1 B): both, or -- for dense plans one tile
  // wide in I (J), 64 x 256 (256 x 64) tiles -- only the short side's A (B): its sums cost
  // nothing, the long side's slots would be 49 x its quadrant (cfg3 at m = 256, L2:
  // 6.6 GB), and a stage of raw long-side views + one slot view leaves room for 3 stages
  int presum_sides = 0;
  // dense-M item order with a tile position's terms consecutive: for problems one
  // tile wide in I or J (cfg3 at m or n = 256), where term-major order re-reads the
  // long operand's views from DRAM once per term (19 GB at 2^24, N_a = 16, L2)
  bool term_inner = false;
  std::vector<int> seq;  // term order of the dense-M batches and accumulate lists
  size_t off_pool = 0, off_vecs = 0, off_tab = 0, off_tickets = 0, off_counters = 0, off_M = 0, off_pa = 0,
         off_pb = 0, off_acc = 0, total = 0;
  size_t off_pool2 = 0, off_const = 0;  // original vectors (repacking); end of the constant region
  std::shared_ptr<Resident> res;        // device snapshots of the constant region
  size_t tab_bytes = 0, acc_bytes = 0;
  int64_t ntickets = 0, ncounters = 0;
  int64_t m_slot = 0, pa_slot = 0, pb_slot = 0;
};

// Workspace cap for the term batches of dense M / operand slots: STC_WORKSPACE_CAP_MB,
// else 40 % of the device's memory (at least 24 GiB; 72 GB on a B200).  A function of
// the device, not of its current free memory, so a re-planned problem gets the same
// workspace size.  The batch count changes no result: each batch's C pass continues
// the previous one's sums in the same order.
int64_t cap_bytes() {
  if (const char *e = stc_env("STC_WORKSPACE_CAP_MB")) return atoll(e) * (int64_t)1024 * 1024;
  const int64_t floor_bytes = (int64_t)24 << 30;
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
    cudaGetLastError();  // no device (planning on a CPU host): clear the error
    return floor_bytes;
  }
  return std::max<int64_t>(floor_bytes, (int64_t)(tot / 10 * 4));
}

// The terms' execution (and C-update) order: the reference's term order
// (strassen.py:173-178), or reordered so that terms running concurrently (within
// `window` consecutive terms) update disjoint C quadrants (fewer ticket waits).
// Measured: the reordering pays on quadrants taller than wide (cfg3 2^24 N_a = 128
// L2, 4096 x 256: 3.63 vs 3.99 ms) and costs 2 % on square / wide ones (cfg2 L2 3.44
// vs 3.38 ms, cfg3 N_a = 32 3.63 vs 3.56 ms), so `windowed` is the caller's choice
// (tall ticketed plans); STC_EXEC_ORDER=reference|windowed forces either.  In the
// reference order the variants add the M products into C as the reference does.
std::vector<int> exec_order(const std::vector<Term> &terms, int window, bool windowed) {
  const int T = (int)terms.size();
  std::vector<int> seq;
  seq.reserve(T);
  if (const char *env = stc_env("STC_EXEC_ORDER")) windowed = strcmp(env, "windowed") == 0;
  if (window <= 1 || !windowed) {
    for (int i = 0; i < T; ++i) seq.push_back(i);
    return seq;
  }
  std::vector<char> used(T, 0);
  for (int step = 0; step < T; ++step) {
    int best = -1;
    long best_score = -1;
    for (int cand = 0; cand < T; ++cand) {
      if (used[cand]) continue;
      long score = 0;  // higher = better: distance-weighted conflicts subtracted
      for (int back = 1; back < window && back <= (int)seq.size(); ++back) {
        const Term &prev = terms[seq[seq.size() - back]];
        for (const Op &x : terms[cand].c)
          for (const Op &y : prev.c)
            if (x.q == y.q) score -= (long)(window - back) * 1000;
      }
      if (best < 0 || score > best_score) {
        best = cand;
        best_score = score;
      }
      if (score == 0) break;  // first conflict-free term in reference order
    }
    used[best] = 1;
    seq.push_back(best);
  }
  return seq;
}

// Operand sides seen by the fused kernel: the original tensors (direct) or
// their repacked quadrant blocks (packed_sides).
struct FusedSides {
  stc_bundle ax, ak, bk, bx;  // A rows (I), A cols (P), B rows (P), B cols (J)
  Tiling tax, tak, tbk, tbx;
  int akf = 0, bkf = 0;
  int64_t a_base = 0, b_base = 0;            // map base offsets (elements)
  int64_t start[4], len[4], vbase[4];        // pool vectors ar, ac, br, bc: start, length, subtracted base
  int64_t qxa = 0, qk = 0, qxb = 0;          // quadrant (or slot) lengths of the A-x, k and B-x bundles
};

struct TmaSide;
bool plan_cred_side(const stc_bundle &rb, const Tiling &tr, const stc_bundle &cb, const Tiling &tc, int level,
                    const double *data, int64_t base, TmaSide &ts);
bool c_boxes_regular(const stc_problem *p, const Tiling &ti, const Tiling &tj, int level);
FusedSides direct_sides(const stc_problem *p, const Plan &pl);
FusedSides packed_sides(const Plan &pl);
FusedSides naive_sides(const Plan &pl);
FusedSides mixed_sides(const stc_problem *p, const Plan &pl);
bool plan_fused(const stc_problem *p, const Plan &pl, const FusedSides &fs, const double *A, const double *B,
                const double *C, GemmArgs &g, CUtensorMap maps[3], CoordJobs &jobs);

// Pre-summed operands for ABC / AB at L = 1, 2, 3 (STC_PRESUM_OPS = 0 / 1 forces it off /
// on).  The sums cost one HBM pass per side (4^L quadrant reads + 7^L slot writes per
// element position) and take every DADD off the FP64 pipe the DMMAs use: the fused
// kernel's in-SM sums cost it 4-10 % (L1; 10 % with A k-contiguous) / 18 % (L2) of its DMMA time (cfg2, 16384^3,
// cfg5; tools/presum_sweep.py).  Operands whose views are not TMA boxes are repacked
// anyway (one read + one write of every quadrant), which the presum pass replaces.
// Cost model at 5 TB/s and 33 TF/s executed.
bool presum_wanted(const stc_problem *p, const Plan &pl) {
  if (pl.level < 1 || pl.level > 3 || pl.variant == STC_VARIANT_NAIVE) return false;
  if (pl.flags & (STC_FLAG_FORCE_SLOW | STC_FLAG_REFERENCE_TILING)) return false;
  if (const char *e = stc_env("STC_FUSED"))
    if (atoi(e) == 0) return false;
  if (const char *e = stc_env("STC_PRESUM_OPS")) return atoi(e) != 0;
  // L = 3: up to 8 views per side are beyond the fused kernel's stages -- without slots the
  // gather kernel runs the problem (16384^3 L3 ABC 562 ms against 208 ms through slots)
  if (pl.level == 3) return true;
  const double qa = (double)pl.mq_pad * pl.kq_pad, qb = (double)pl.kq_pad * pl.nq_pad;
  const double quads = (double)pl.nquads, T = pl.level == 1 ? 7.0 : 49.0;
  const double t_presum = 8.0 * (quads + T) * (qa + qb) / 5e12;
  GemmArgs g{};
  CUtensorMap maps[3];
  CoordJobs jobs{};
  const bool direct = plan_fused(p, pl, direct_sides(p, pl), nullptr, nullptr, nullptr, g, maps, jobs);
  const double t_repack = direct ? 0.0 : 8.0 * 2.0 * quads * (qa + qb) / 3e12;  // gathers: ~50 % of HBM
  const double t_gemm = T * 2.0 * (double)pl.mq_pad * pl.nq_pad * pl.kq_pad / 33e12;
  const double penalty = pl.level == 1 ? 0.10 : 0.18;
  return t_presum < penalty * t_gemm + t_repack;
}

int build_plan(const stc_problem *p, Plan &pl, int grid_hint) {
  if (!p) return fail(STC_EINVAL, "null problem");
  const char *names[6] = {"a_row", "a_col", "b_row", "b_col", "c_row", "c_col"};
  const stc_bundle *bs[6] = {&p->a_row, &p->a_col, &p->b_row, &p->b_col, &p->c_row, &p->c_col};
  for (int i = 0; i < 6; ++i)
    if (int rc = check_bundle(*bs[i], names[i])) return rc;
  if (!same_extents(p->a_row, p->c_row)) return fail(STC_EINVAL, "I bundle extents of A and C differ");
  if (!same_extents(p->a_col, p->b_row)) return fail(STC_EINVAL, "P bundle extents of A and B differ");
  if (!same_extents(p->b_col, p->c_col)) return fail(STC_EINVAL, "J bundle extents of B and C differ");
  if (p->level < 0) return fail(STC_EINVAL, "level must be non-negative, got %d", p->level);
  if ((1 << p->level) > MAX_OPS)
    return fail(STC_ECAP, "level %d exceeds the device cap of %d", p->level, 4);
  if (p->variant < 0 || p->variant > 2) return fail(STC_EINVAL, "unknown variant %d", p->variant);
  pl.level = p->level;
  pl.variant = p->variant;
  pl.flags = p->flags;
  pl.m = bundle_len(p->a_row);
  pl.k = bundle_len(p->a_col);
  pl.n = bundle_len(p->b_col);
  pl.Q = (int64_t)1 << pl.level;
  pl.nquads = (int)(pl.Q * pl.Q);
  pl.mq = cdiv(pl.m, pl.Q);
  pl.nq = cdiv(pl.n, pl.Q);
  pl.kq = cdiv(pl.k, pl.Q);
  // tile orders per bundle (see make_tiling)
  const bool ref = (p->flags & STC_FLAG_REFERENCE_TILING) != 0;
  const int a_min = min_stride_side(p->a_row, p->a_col);
  const int b_min = min_stride_side(p->b_row, p->b_col);
  const int c_min = min_stride_side(p->c_row, p->c_col);
  const int64_t *key_i = a_min == 0 ? p->a_row.str : (c_min == 0 ? p->c_row.str : p->a_row.str);
  const int64_t *key_j = b_min == 1 ? p->b_col.str : (c_min == 1 ? p->c_col.str : p->b_col.str);
  const int64_t *key_p = a_min == 1 ? p->a_col.str : (b_min == 0 ? p->b_row.str : p->a_col.str);
  const Tiling ti = make_tiling(p->a_row, pl.level, key_i, ref);
  const Tiling tj = make_tiling(p->b_col, pl.level, key_j, ref);
  const Tiling tp = make_tiling(p->a_col, pl.level, key_p, ref);
  // CTA tile shape: 64 x 256 (256 x 64) when the I (J) quadrants are at most 64 past a
  // multiple of 128 -- a 128-row tile would be half padding -- for the dense-M launches
  // with the summing warpgroup (AB, ABC with such C tiles, L >= 1); see shape_usable
  pl.tshape = 0;
  const int req_shape = p->tiling & 0xf, req_stages = (p->tiling >> 4) & 0xf;
  if ((p->tiling & ~0xff) != 0 || req_shape > 5 || req_stages == 1)
    return fail(STC_EINVAL, "tiling 0x%x: shape must be 0..5 (1 + CTA tile shape), stages 0 or 2..15", p->tiling);
  pl.stage_cap = req_stages;
  {
    const char *ts = stc_env("STC_TSHAPE");
    // (A / B base offsets even: TMA needs 16-byte aligned views of the 256-byte aligned
    // allocations; the shaped plan has no gather-kernel fallback)
    // (L >= 3 runs on the fused kernel only through pre-summed slots: L = 3 unless switched off)
    const bool deep_gather = pl.level > 3 || (pl.level == 3 && stc_env("STC_PRESUM_OPS") && atoi(stc_env("STC_PRESUM_OPS")) == 0);
    const bool allowed = (!ts || atoi(ts) != 0) && pl.level >= 1 && !deep_gather && pl.variant != STC_VARIANT_NAIVE &&
                         p->a_base % 2 == 0 && p->b_base % 2 == 0 &&
                         !(p->flags & (STC_FLAG_FORCE_SLOW | STC_FLAG_REFERENCE_TILING)) &&
                         !(stc_env("STC_FUSED") && atoi(stc_env("STC_FUSED")) == 0) &&
                         !(stc_env("STC_PRESUM") && atoi(stc_env("STC_PRESUM")) != 1) &&
                         !(pl.variant == STC_VARIANT_ABC && stc_env("STC_ABC_DENSE") && atoi(stc_env("STC_ABC_DENSE")) == 0);
    // the shape with the least padded area (128 x 128 on ties): cfg4 L2 (1138 x 788
    // quadrants) keeps 128 x 128 (87 % useful) over 256 x 64 (84 %)
    const int64_t a0 = rup(pl.mq, BM) * rup(pl.nq, BN), a1 = rup(pl.mq, 64) * rup(pl.nq, 256),
                  a2 = rup(pl.mq, 256) * rup(pl.nq, 64);
    const int64_t a4 = rup(pl.mq, BM) * rup(pl.nq, 64);
    // (shape 4, 128 x 64: dense-M plans only -- AB, Naive slots excluded above, ABC whose C
    // tiles are not TMA-reduce boxes -- with at least 15 % less padded area: its 32 x 32
    // warp tiles cost ~7 % per flop, cfg4 L2's 7 % less padding bought nothing; cfg1 L2
    // (144-wide quadrants, 25 % less) 50.7 -> 48.7 us)
    const bool dense_anyway = pl.variant != STC_VARIANT_ABC || !c_boxes_regular(p, ti, tj, pl.level);
    if (allowed && pl.mq % BM != 0 && pl.mq % BM <= 64 && pl.nq >= 256 && a1 < a0) pl.tshape = 1;
    else if (allowed && pl.nq % BN != 0 && pl.nq % BN <= 64 && pl.mq >= 256 && a2 < a0) pl.tshape = 2;
    else if (allowed && dense_anyway && (double)a4 <= 0.85 * (double)a0) pl.tshape = 4;
    // shape 3 (64 x 128, 32 x 32 warp tiles): for problems of a few waves, when its
    // waves x tile area -- the per-SM work in sequence -- is clearly below the chosen
    // shape's (cfg1 L1: 105 items in one wave instead of 70; L2: 294 items in two waves
    // instead of 196 in two of twice the work).  Dense M output (grid >= 4 tiles per term).
    const int64_t T = (int64_t)std::pow(7.0, pl.level), grid = grid_hint > 0 ? grid_hint : 148;
    const int64_t tm0 = pl.tshape == 1 ? 64 : pl.tshape == 2 ? 256 : BM,
                  tn0 = pl.tshape == 1 ? 256 : pl.tshape == 2 || pl.tshape == 4 ? 64 : BN;
    const int64_t p_cur = cdiv(pl.mq, tm0) * cdiv(pl.nq, tn0), p3 = cdiv(pl.mq, 64) * cdiv(pl.nq, 128);
    const int64_t waves_cur = cdiv(T * p_cur, grid), waves3 = cdiv(T * p3, grid);
    if (allowed && T > 1 && grid >= 4 * p3 && waves_cur <= 4 &&
        (double)waves3 * 64 * 128 < 0.85 * (double)waves_cur * tm0 * tn0)
      pl.tshape = 3;
    if (allowed && ts && atoi(ts) > 0 && atoi(ts) <= 4) pl.tshape = atoi(ts);  // forced (diagnostics)
    if (req_shape > 0) {  // the caller's tile config (stc_problem.tiling)
      if (req_shape - 1 != 0 && !allowed)
        return fail(STC_EINVAL, "tile shape %d needs L >= 1, a non-Naive variant, even A / B base offsets and "
                    "no force_slow / reference tiling", req_shape - 1);
      pl.tshape = req_shape - 1;
    }
  }
  pl.tm = pl.tshape == 1 || pl.tshape == 3 ? 64 : pl.tshape == 2 ? 256 : BM;
  pl.tn = pl.tshape == 1 ? 256 : pl.tshape == 2 || pl.tshape == 4 ? 64 : pl.tshape == 3 ? 128 : BN;
  pl.mq_pad = rup(pl.mq, pl.tm);
  pl.nq_pad = rup(pl.nq, pl.tn);
  pl.kq_pad = rup(pl.kq, BK);

  pl.ti = ti;
  pl.tj = tj;
  pl.tp = tp;
  pl.a_kfast = a_min == 1;
  pl.b_kfast = b_min == 0;
  if (!stc_env("STC_NO_USTEP")) {
    pl.a_ustep = pl.a_kfast ? unit_step(p->a_col, tp, rup(pl.kq, BK), pl.a_ugroup)
                            : unit_step(p->a_row, ti, rup(pl.mq, pl.tm), pl.a_ugroup);
    pl.b_ustep = pl.b_kfast ? unit_step(p->b_row, tp, rup(pl.kq, BK), pl.b_ugroup)
                            : unit_step(p->b_col, tj, rup(pl.nq, pl.tn), pl.b_ugroup);
  }
  if (pl.tshape != 0) {  // the direct fused layout must cut the new tiles as boxes -- or the
    GemmArgs gd{};      // operands come from pre-summed slots, box-regular by construction
    CUtensorMap md[3];
    CoordJobs jd{};
    if (!plan_fused(p, pl, direct_sides(p, pl), nullptr, nullptr, nullptr, gd, md, jd) && !presum_wanted(p, pl)) {
      if (req_shape > 0)
        return fail(STC_EINVAL, "tile shape %d: the operand views cannot be cut into its TMA boxes", req_shape - 1);
      pl.tshape = 0;
      pl.tm = BM;
      pl.tn = BN;  // (the dense / ticketed choice below sees the 128 x 128 tiles)
      pl.mq_pad = rup(pl.mq, BM);
      pl.nq_pad = rup(pl.nq, BN);
    }
  }

  // pool vectors (subsystem 1)
  auto add = [&](VecDesc d) {
    d.out_start = pl.pool_len;
    pl.pool_len += d.nq * d.q_len_pad;
    pl.vecs.push_back(d);
    return d.out_start;
  };
  pl.ar = add(vec_bundle(p->a_row, 0, pl.Q, pl.tm, ti));
  pl.ac = add(vec_bundle(p->a_col, p->a_base, pl.Q, BK, tp));
  pl.br = add(vec_bundle(p->b_row, 0, pl.Q, BK, tp));
  pl.bc = add(vec_bundle(p->b_col, p->b_base, pl.Q, pl.tn, tj));
  pl.cr = add(vec_bundle(p->c_row, 0, pl.Q, pl.tm, ti));
  pl.cc = add(vec_bundle(p->c_col, p->c_base, pl.Q, pl.tn, tj));

  pl.terms = strassen_terms(pl.level);
  for (const Term &t : pl.terms) pl.max_ops = std::max(pl.max_ops, (int)std::max(t.a.size(), t.b.size()));
  const int T = (int)pl.terms.size();
  const int64_t P = (pl.mq_pad / pl.tm) * (pl.nq_pad / pl.tn);
  if (P * (int64_t)T > INT32_MAX) return fail(STC_EINVAL, "problem too large: %lld work items", (long long)(P * T));
  pl.grid = grid_hint > 0 ? grid_hint : 148;

  pl.seq.resize(T);
  for (int t = 0; t < T; ++t) pl.seq[t] = t;
  if (pl.variant == STC_VARIANT_ABC) {
    // C-tile update order (tickets, or the dense-M accumulate order): terms
    // that run concurrently should write disjoint quadrants
    // (window from the 128 x 128 tile count: every tile shape and operand path of a
    // problem gets the same C-update order, so their results stay bitwise equal)
    const int64_t P128 = cdiv(pl.mq, BM) * cdiv(pl.nq, BN);
    const int window = (int)std::min<int64_t>(T, cdiv(pl.grid, P128) + 1);
    pl.seq = exec_order(pl.terms, window, cdiv(pl.mq, BM) > cdiv(pl.nq, BN));
    // dense-M mode when many terms per C tile would be in flight at once: the
    // ticket chains then serialise (cfg2 pieces of m = 1024: 9 terms in flight,
    // 1.56 ms ticketed vs 1.21 ms dense; 576^3 L2: 0.60 vs 0.15 ms).
    // STC_ABC_DENSE = 0 / 1 forces either.
    // Also when the C targets are not regular boxes: the kernel's C updates would then
    // be load/add/store scatters in the consumers (cfg4 L2: 5.2 ms ticketed, 3.2 dense).
    const char *de = stc_env("STC_ABC_DENSE");
    // (the shaped tiles 1-4 write dense M only)
    const bool dense = T > 1 && (de ? atoi(de) != 0
                                    : (pl.grid >= 4 * P || pl.tshape != 0 ||
                                       !c_boxes_regular(p, pl.ti, pl.tj, pl.level)));
    pl.ticketed = !dense;
  }
  {
    const char *ti_env = stc_env("STC_TERM_INNER");
    const bool skinny = pl.mq_pad / pl.tm == 1 || pl.nq_pad / pl.tn == 1;
    pl.term_inner = !pl.ticketed && T > 1 && (ti_env ? atoi(ti_env) != 0 : skinny);
  }
  // Operand sums pre-formed into per-term slots (k_presum): ABC and AB when worth it
  // (AB with pre-summed operands is the Naive schedule: the same M products), and
  // always for Naive (its explicit submatrix copies) at L <= 3 (k_unpack beyond).
  pl.presum = pl.variant == STC_VARIANT_NAIVE ? (pl.level >= 1 && pl.level <= 3) : presum_wanted(p, pl);
  pl.presum_sides = pl.presum ? 3 : 0;
  if (pl.variant != STC_VARIANT_NAIVE && !pl.ticketed && pl.level >= 1 && pl.level <= 2 &&
      !(pl.flags & (STC_FLAG_FORCE_SLOW | STC_FLAG_REFERENCE_TILING)) &&
      bundle_len(p->a_col) == pl.Q * pl.kq_pad) {  // (the direct side's k quadrants need no padding)
    const char *e = stc_env("STC_PRESUM_SIDES");  // 1 / 2 / 3 force (diagnostics), 0 disables one-sided
    const int want = e ? (atoi(e) & 3) : stc_env("STC_PRESUM_OPS") ? 0 : pl.tshape == 1 ? 1 : pl.tshape == 2 ? 2 : 0;
    if (want == 3) {
      pl.presum = true;
      pl.presum_sides = 3;
    } else if (want == 1 || want == 2) {
      const bool was = pl.presum;
      const int was_sides = pl.presum_sides;
      pl.presum = true;
      pl.presum_sides = want;
      GemmArgs gx{};
      CUtensorMap mx[3];
      CoordJobs jx{};
      if (!plan_fused(p, pl, mixed_sides(p, pl), nullptr, nullptr, nullptr, gx, mx, jx)) {
        pl.presum = was;  // the long side's own views are not boxes: keep the default
        pl.presum_sides = was_sides;
      }
    }
  }
  const bool slots = pl.variant == STC_VARIANT_NAIVE || pl.presum;
  if (slots) {
    // per-term slots of packed operand sums, oriented like the source (unit stride in
    // k -> [x][k] slots, else [k][x]) so both sides of the copy coalesce
    const bool all = pl.variant == STC_VARIANT_NAIVE || pl.presum_sides == 3;  // (Naive: k_presum or k_unpack)
    pl.pa_slot = all || (pl.presum_sides & 1) ? pl.kq_pad * pl.mq_pad : 0;
    pl.pb_slot = all || (pl.presum_sides & 2) ? pl.kq_pad * pl.nq_pad : 0;
    pl.m_slot = pl.ticketed ? 0 : pl.mq_pad * pl.nq_pad;
    int64_t b = cap_bytes() / std::max<int64_t>((pl.pa_slot + pl.pb_slot + pl.m_slot) * 8, 1);
    pl.batch = (int)std::max<int64_t>(1, std::min<int64_t>(b, T));
    pl.nbatches = (int)cdiv(T, pl.batch);
    pl.dka = add(vec_affine(pl.kq_pad, pl.kq_pad, pl.a_kfast ? 1 : pl.mq_pad));
    pl.dkb = add(vec_affine(pl.kq_pad, pl.kq_pad, pl.b_kfast ? 1 : pl.nq_pad));
    pl.dxa = add(slot_vec(pl.mq_pad, pl.a_kfast ? pl.kq_pad : 1, pl.pa_slot, pl.batch));
    pl.dxb = add(slot_vec(pl.nq_pad, pl.b_kfast ? pl.kq_pad : 1, pl.pb_slot, pl.batch));
  }
  if (pl.ticketed) {
    const std::vector<int> &seq = pl.seq;
    std::vector<int> writers(pl.nquads, 0);
    for (int t : seq) {
      const Term &tm = pl.terms[t];
      TermDesc d{};
      d.a_first = (int)pl.ops.size();
      d.a_count = (int)tm.a.size();
      for (const Op &o : tm.a) {
        int64_t r, c;
        quad_rc(o.q, pl.level, r, c);
        pl.ops.push_back({pl.ar + r * pl.mq_pad, pl.ac + c * pl.kq_pad, 0, (double)o.s});
      }
      d.b_first = (int)pl.ops.size();
      d.b_count = (int)tm.b.size();
      for (const Op &o : tm.b) {
        int64_t r, c;
        quad_rc(o.q, pl.level, r, c);
        pl.ops.push_back({pl.bc + c * pl.nq_pad, pl.br + r * pl.kq_pad, 0, (double)o.s});
      }
      d.c_first = (int)pl.tgts.size();
      d.c_count = (int)tm.c.size();
      for (const Op &o : tm.c) {
        int64_t r, c;
        quad_rc(o.q, pl.level, r, c);
        TgtDesc g{};
        g.row_start = pl.cr + r * pl.mq_pad;
        g.col_start = pl.cc + c * pl.nq_pad;
        g.sign = (double)o.s;
        g.ticket_base = (int32_t)(o.q * P);
        g.order = writers[o.q]++;
        pl.tgts.push_back(g);
      }
      d.m_slot = t;
      pl.tdesc.push_back(d);
    }
    pl.ntickets = (int64_t)pl.nquads * P;
    if (pl.presum) {
      // one view per side: the term's slot of pre-summed operands (batch-local slot
      // t % batch of the exec-order position t; the batches run one launch each)
      pl.ops.clear();
      for (int s = 0; s < pl.batch; ++s) {
        pl.ops.push_back({pl.dxa + s * pl.mq_pad, pl.dka, 0, 1.0});
        pl.ops.push_back({pl.dxb + s * pl.nq_pad, pl.dkb, 0, 1.0});
      }
      for (int t = 0; t < T; ++t) {
        TermDesc &d = pl.tdesc[t];
        d.a_first = 2 * (t % pl.batch);
        d.b_first = d.a_first + 1;
        d.a_count = d.b_count = 1;
      }
      pl.ncounters = pl.nbatches;
    } else {
      pl.batch = T;
      pl.nbatches = 1;
      pl.ncounters = 1;
    }
  } else {
    // dense M slots (and the packed operand slots above), batched under the cap
    pl.m_slot = pl.mq_pad * pl.nq_pad;
    if (!slots) {
      int64_t b = cap_bytes() / std::max<int64_t>(pl.m_slot * 8, 1);
      pl.batch = (int)std::max<int64_t>(1, std::min<int64_t>(b, T));
      pl.nbatches = (int)cdiv(T, pl.batch);
    }
    pl.ncounters = pl.nbatches;
  }

  // fused kernel on repacked operands when the views are not box-regular
  if (!slots) {
    GemmArgs gd{};
    CUtensorMap md[3];
    CoordJobs jd{};
    const bool direct = plan_fused(p, pl, direct_sides(p, pl), nullptr, nullptr, nullptr, gd, md, jd);
    pl.need_pack = !direct && plan_fused(p, pl, packed_sides(pl), nullptr, nullptr, nullptr, gd, md, jd) &&
                   !(stc_env("STC_PACK") && atoi(stc_env("STC_PACK")) == 0);
  }
  if (pl.ticketed) {
    pl.tab_bytes = pl.tdesc.size() * sizeof(TermDesc) + pl.ops.size() * sizeof(OpDesc) + pl.tgts.size() * sizeof(TgtDesc);
  } else {
    // per batch: TermDesc[batch] + OpDesc (<= 2*Q per side per term) + accumulate lists
    const size_t ops_max = (size_t)pl.batch * 2 * (size_t)(pl.Q * 2 + 2);
    pl.tab_bytes = (size_t)pl.batch * sizeof(TermDesc) * 3 + ops_max * sizeof(OpDesc);
    pl.acc_bytes = align256((size_t)(pl.nquads + 1) * 4) + align256((size_t)pl.batch * pl.nquads * 4) +
                   align256((size_t)pl.batch * pl.nquads * 8) + 2 * align256((size_t)pl.nquads * 8);
  }

  // workspace layout: the constant region first (the per-plan snapshot, Resident), then
  // the per-call buffers
  size_t off = 0;
  pl.off_pool = off;
  off = align256(off + (size_t)pl.pool_len * 8);
  pl.off_pool2 = off;  // the original vectors while `pool` holds the repacked ones
  if (pl.need_pack) off = align256(off + (size_t)pl.pool_len * 8);
  pl.off_kbs = off;
  off = align256(off + (size_t)(pl.pool_len / BK) * 8);
  pl.off_coords = off;  // fused kernel: int4 map coordinates per 8 pool entries
  off = align256(off + (size_t)(pl.pool_len / 8) * 16);
  pl.off_vecs = off;
  off = align256(off + (pl.vecs.size() + 4) * sizeof(VecDesc));  // + the packed sides' vectors
  pl.off_tab = off;
  off = align256(off + pl.tab_bytes * (pl.ticketed ? 1 : pl.nbatches));
  pl.off_acc = off;
  off = align256(off + pl.acc_bytes * (pl.ticketed ? 0 : pl.nbatches));
  pl.off_tickets = off;
  off = align256(off + (size_t)pl.ntickets * 4);
  pl.off_counters = off;
  off = align256(off + (size_t)pl.ncounters * 4);
  pl.off_const = off;
  pl.off_mscr = off;  // fused ABC: EPI_BUFS M tiles per CTA for the epilogue warps
  if (pl.ticketed) off = align256(off + (size_t)pl.grid * EPI_BUFS * BM * BN * 8);
  pl.off_pka = off;
  if (pl.need_pack) off = align256(off + (size_t)(pl.Q * pl.Q) * pl.mq_pad * pl.kq_pad * 8);
  pl.off_pkb = off;
  if (pl.need_pack) off = align256(off + (size_t)(pl.Q * pl.Q) * pl.nq_pad * pl.kq_pad * 8);
  pl.off_M = off;
  if (!pl.ticketed) off = align256(off + (size_t)pl.batch * pl.m_slot * 8);
  pl.off_pa = off;
  if (slots) off = align256(off + (size_t)pl.batch * pl.pa_slot * 8);
  pl.off_pb = off;
  if (slots) off = align256(off + (size_t)pl.batch * pl.pb_slot * 8);
  pl.res = std::make_shared<Resident>();
  pl.total = off;
  return STC_OK;
}


// ------------------------------------------------------------ TMA staging
// A side (A or B) can be staged with tensor-map box loads when every unit --
// one view's 128-row tile x one 16-deep k-chunk -- is a box of the tensor:
// the bundles' tile orders (make_tiling) cut tiles and chunks as aligned
// sub-boxes, the tensor's unit-stride label leads the tile order of its
// bundle, and the strides meet TMA's rules.  The map's dims are then ordered
// so that the box lands as raw[k][128] (unit stride in x) or raw[x][16] (unit
// stride in k, 16-element rows swizzled).  Otherwise the side uses the
// cp.async gather (always correct; the reference's fast/slow split,
// _jit.py:54-78, becomes TMA vs gather).
struct TmaSide {
  int rank = 0;
  cuuint64_t dims[5];
  cuuint64_t strides[4];  // bytes, dims 1..rank-1
  cuuint32_t box[5];
  int src[5];
  int np[2] = {0, 0};
  int64_t pstr[2][4];
  int swizzle = 0;  // 0, 64 or 128 (bytes)
};

// Merge tensor-map dims that address one contiguous run of elements (TMA allows
// 5): a dim j whose stride is dim i's stride x extent (same part) folds into i when
// j's box is 1 (the box along i is unchanged) or when j directly follows i and i's
// box covers its whole extent (the boxes concatenate; smem layout unchanged).  Dim 0
// keeps its box (the swizzle span bounds the inner box).  cfg5's A[a,b,c,e,f,g]:
// (g, f, e) and (c, b, a) are each one dim.
template <class D>
void merge_dims(std::vector<D> &dims) {
  for (bool changed = true; changed;) {
    changed = false;
    for (size_t i = 0; i < dims.size() && !changed; ++i)
      for (size_t j = 0; j < dims.size() && !changed; ++j) {
        if (i == j || dims[i].isx != dims[j].isx || dims[j].str != dims[i].str * dims[i].ext) continue;
        const bool fold = dims[j].box == 1;
        const bool concat = i > 0 && j == i + 1 && dims[i].box == dims[i].ext;
        if (!fold && !concat) continue;
        if (concat) dims[i].box *= dims[j].box;
        dims[i].ext *= dims[j].ext;
        dims.erase(dims.begin() + j);
        changed = true;
      }
  }
}

// Tile sub-box of a bundle: per label, the extent covered by one tile of
// `tile` consecutive tile-order indices, and the labels in tile order.
bool tile_subbox(const stc_bundle &b, const Tiling &t, int64_t tile, int64_t *tb, int *ord, int &nord) {
  for (int d = 0; d < b.nlab; ++d) tb[d] = 1;
  nord = 0;
  int64_t rem = tile;
  for (int j = 0; j < t.nbox && rem > 1; ++j) {
    const int d = t.order[j];
    const int64_t e = t.box_ext[d];
    if (e == 1) continue;
    if (rem >= e) {
      if (rem % e) return false;
      tb[d] = e;
      rem /= e;
    } else {
      if (e % rem) return false;
      tb[d] = rem;
      rem = 1;
    }
    ord[nord++] = d;
  }
  return rem == 1;
}

bool plan_tma_side(const stc_bundle &xb, const Tiling &tx, const stc_bundle &kb, const Tiling &tk, int level, int kfast,
                   const double *data, int64_t base, TmaSide &ts) {
  if (tx.nbox == 0 || tk.nbox == 0) return false;
  const int64_t Q = (int64_t)1 << level;
  if ((bundle_len(xb) / Q) % BM != 0 || (bundle_len(kb) / Q) % BK != 0) return false;
  int64_t tbx[STC_MAX_LABELS], tbk[STC_MAX_LABELS];
  int ox[STC_MAX_LABELS], ok_[STC_MAX_LABELS], nox = 0, nok = 0;
  if (!tile_subbox(xb, tx, BM, tbx, ox, nox) || !tile_subbox(kb, tk, BK, tbk, ok_, nok)) return false;
  // map dims: the leading part (unit-stride side) in tile order, the other part, then box-1 labels
  struct Dim {
    int64_t ext, str, box;
    bool isx;
    int lab;
  };
  std::vector<Dim> dims;
  auto push_ordered = [&](const stc_bundle &b, const int64_t *tb, const int *ord, int n, bool isx) {
    for (int j = 0; j < n; ++j) dims.push_back({b.ext[ord[j]], b.str[ord[j]], tb[ord[j]], isx, ord[j]});
  };
  if (kfast) {
    push_ordered(kb, tbk, ok_, nok, false);
    push_ordered(xb, tbx, ox, nox, true);
  } else {
    push_ordered(xb, tbx, ox, nox, true);
    push_ordered(kb, tbk, ok_, nok, false);
  }
  for (int pass = 0; pass < 2; ++pass) {
    const stc_bundle &b = pass == 0 ? xb : kb;
    const int64_t *tb = pass == 0 ? tbx : tbk;
    for (int d = 0; d < b.nlab; ++d)
      if (b.ext[d] > 1 && tb[d] == 1) dims.push_back({b.ext[d], b.str[d], 1, pass == 0, d});
  }
  merge_dims(dims);
  if (dims.empty() || dims.size() > 5) return false;
  if (dims[0].str != 1) return false;                          // unit stride leads the box
  if (kfast && dims[0].box != BK) return false;                // one swizzled 128-byte row per x
  if (!kfast && (dims[0].box * 8) % 16 != 0) return false;
  for (size_t d = 0; d < dims.size(); ++d) {
    if (dims[d].str <= 0 || dims[d].box > 256 || dims[d].ext >= (int64_t)1 << 31) return false;
    if (d > 0 && ((dims[d].str % 2) != 0 || dims[d].str * 8 >= ((int64_t)1 << 40))) return false;
  }
  if ((reinterpret_cast<uintptr_t>(data + base) & 15) != 0) return false;
  // coordinate parts: labels of each bundle by descending stride, strides nested
  for (int part = 0; part < 2; ++part) {
    std::vector<int> idx;
    for (size_t d = 0; d < dims.size(); ++d)
      if (dims[d].isx == (part == 0)) idx.push_back((int)d);
    if (idx.empty() || idx.size() > 4) return false;
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return dims[a].str > dims[b].str; });
    for (size_t i = 0; i + 1 < idx.size(); ++i)
      if (dims[idx[i]].str < dims[idx[i + 1]].str * dims[idx[i + 1]].ext) return false;
    ts.np[part] = (int)idx.size();
    for (size_t i = 0; i < idx.size(); ++i) {
      ts.pstr[part][i] = dims[idx[i]].str;
      ts.src[idx[i]] = part * 4 + (int)i;
    }
    for (size_t i = idx.size(); i < 4; ++i) ts.pstr[part][i] = 1;
  }
  ts.rank = (int)dims.size();
  for (int d = 0; d < ts.rank; ++d) {
    ts.dims[d] = (cuuint64_t)dims[d].ext;
    ts.box[d] = (cuuint32_t)dims[d].box;
    if (d > 0) ts.strides[d - 1] = (cuuint64_t)(dims[d].str * 8);
  }
  for (int d = ts.rank; d < 5; ++d) ts.src[d] = 0;
  ts.swizzle = kfast ? 128 : 0;
  return true;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool encode_side(const TmaSide &ts, const double *data, int64_t base, CUtensorMap &map) {
  PFN_cuTensorMapEncodeTiled_v12000 fn = encode_fn();
  if (!fn) return false;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  if (const char *e = stc_env("STC_TMA_PROMO"))
    promo = atoi(e) == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
            : atoi(e) == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
            : atoi(e) == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  const CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)ts.rank, (void *)(data + base), ts.dims,
                        ts.strides, ts.box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        ts.swizzle == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : ts.swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Both sides of the operand views of `p` (A: I x P, B: P x J) as tensor maps;
// false (gather path) unless both qualify.  STC_TMA=0 disables.
bool plan_tma(const stc_problem *p, const Plan &pl, const double *A, const double *B, GemmArgs &g, CUtensorMap maps[2]) {
  if (const char *e = stc_env("STC_TMA"))
    if (atoi(e) == 0) return false;
  if (pl.flags & (STC_FLAG_FORCE_SLOW | STC_FLAG_REFERENCE_TILING)) return false;
  TmaSide sa, sb;
  if (!plan_tma_side(p->a_row, pl.ti, p->a_col, pl.tp, pl.level, pl.a_kfast, A, p->a_base, sa)) return false;
  if (!plan_tma_side(p->b_col, pl.tj, p->b_row, pl.tp, pl.level, pl.b_kfast, B, p->b_base, sb)) return false;
  int nraw = 0, kwin = 0;
  if (!gemm_tma_config(pl.max_ops, nraw, kwin)) return false;
  if (!encode_side(sa, A, p->a_base, maps[0]) || !encode_side(sb, B, p->b_base, maps[1])) return false;
  const TmaSide *ss[2] = {&sa, &sb};
  for (int sd = 0; sd < 2; ++sd) {
    g.tm_rank[sd] = ss[sd]->rank;
    for (int d = 0; d < 5; ++d) g.tm_src[sd][d] = ss[sd]->src[d];
    for (int part = 0; part < 2; ++part) {
      g.tm_np[sd][part] = ss[sd]->np[part];
      for (int i = 0; i < 4; ++i) g.tm_pstr[sd][part][i] = ss[sd]->pstr[part][i];
    }
  }
  // which pool vector carries the tensor's base offset (build_plan: ac for A, bc for B)
  g.tm_base[0][0] = 0;
  g.tm_base[0][1] = p->a_base;
  g.tm_base[1][0] = p->b_base;
  g.tm_base[1][1] = 0;
  g.tma = 1;
  // prefetch distance: what the k-coordinate window keeps ready (KWIN/2 chunks minus the issue lookahead)
  int pf = std::min(16, (kwin / 2 - 2) * 2);
  if (const char *e = stc_env("STC_TMA_PF")) pf = atoi(e);
  g.tma_prefetch = std::max(0, pf);
  g.nraw = nraw;
  g.kwin = kwin;
  return true;
}


// ---- fused kernel (stc_fused.cu) -----------------------------------------------
// Same regularity conditions as plan_tma_side, for 128 x 8 views whose boxes
// land in the fused kernel's swizzled layouts: unit stride in x -> dims
// (x_lo 16, k..., x_hi...), 128-byte swizzle; unit stride in k -> dims
// (k 8, x...), 64-byte swizzle.  The unit-stride label is split into a 16-wide
// low dim and a high dim when its tile extent exceeds 16.
constexpr int kFusedK = 8;

bool plan_fused_side(const stc_bundle &xb, const Tiling &tx, const stc_bundle &kb, const Tiling &tk, int64_t qx,
                     int64_t qk, int kfast, const double *data, int64_t base, TmaSide &ts, int64_t tile) {
  if (tx.nbox == 0 || tk.nbox == 0) return false;
  if (qx % tile != 0 || qk % BK != 0) return false;  // quadrants cut into whole tiles / chunks
  int64_t tbx[STC_MAX_LABELS], tbk[STC_MAX_LABELS];
  int ox[STC_MAX_LABELS], ok_[STC_MAX_LABELS], nox = 0, nok = 0;
  if (!tile_subbox(xb, tx, tile, tbx, ox, nox) || !tile_subbox(kb, tk, kFusedK, tbk, ok_, nok)) return false;
  struct Dim {
    int64_t ext, str, box;
    bool isx;
  };
  std::vector<Dim> dims;
  if (kfast) {
    if (nok == 0 || kb.str[ok_[0]] != 1 || tbk[ok_[0]] != kFusedK) return false;
    for (int j = 0; j < nok; ++j) dims.push_back({kb.ext[ok_[j]], kb.str[ok_[j]], tbk[ok_[j]], false});
    for (int j = 0; j < nox; ++j) dims.push_back({xb.ext[ox[j]], xb.str[ox[j]], tbx[ox[j]], true});
  } else {
    if (nox == 0 || xb.str[ox[0]] != 1) return false;
    const int64_t e0 = xb.ext[ox[0]], b0 = tbx[ox[0]];
    if (b0 < 16 || b0 % 16 != 0 || (b0 > 16 && e0 % 16 != 0)) return false;
    dims.push_back({b0 > 16 ? 16 : e0, 1, 16, true});
    for (int j = 0; j < nok; ++j) dims.push_back({kb.ext[ok_[j]], kb.str[ok_[j]], tbk[ok_[j]], false});
    if (b0 > 16) dims.push_back({e0 / 16, 16, b0 / 16, true});
    for (int j = 1; j < nox; ++j) dims.push_back({xb.ext[ox[j]], xb.str[ox[j]], tbx[ox[j]], true});
  }
  for (int pass = 0; pass < 2; ++pass) {
    const stc_bundle &b = pass == 0 ? xb : kb;
    const int64_t *tb = pass == 0 ? tbx : tbk;
    for (int d = 0; d < b.nlab; ++d)
      if (b.ext[d] > 1 && tb[d] == 1) dims.push_back({b.ext[d], b.str[d], 1, pass == 0});
  }
  merge_dims(dims);
  if (dims.empty() || dims.size() > 5) return false;
  for (size_t d = 0; d < dims.size(); ++d) {
    if (dims[d].str <= 0 || dims[d].box > 256 || dims[d].ext >= (int64_t)1 << 31) return false;
    if (d > 0 && ((dims[d].str % 2) != 0 || dims[d].str * 8 >= ((int64_t)1 << 40))) return false;
  }
  if (data && (reinterpret_cast<uintptr_t>(data + base) & 15) != 0) return false;
  for (int part = 0; part < 2; ++part) {
    std::vector<int> idx;
    for (size_t d = 0; d < dims.size(); ++d)
      if (dims[d].isx == (part == 0)) idx.push_back((int)d);
    if (idx.empty() || idx.size() > 4) return false;
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return dims[a].str > dims[b].str; });
    for (size_t i = 0; i + 1 < idx.size(); ++i)
      if (dims[idx[i]].str < dims[idx[i + 1]].str * dims[idx[i + 1]].ext) return false;
    ts.np[part] = (int)idx.size();
    for (size_t i = 0; i < idx.size(); ++i) {
      ts.pstr[part][i] = dims[idx[i]].str;
      ts.src[idx[i]] = part * 4 + (int)i;
    }
    for (size_t i = idx.size(); i < 4; ++i) ts.pstr[part][i] = 1;
  }
  ts.rank = (int)dims.size();
  for (int d = 0; d < ts.rank; ++d) {
    ts.dims[d] = (cuuint64_t)dims[d].ext;
    ts.box[d] = (cuuint32_t)dims[d].box;
    if (d > 0) ts.strides[d - 1] = (cuuint64_t)(dims[d].str * 8);
  }
  for (int d = ts.rank; d < 5; ++d) ts.src[d] = 0;
  ts.swizzle = kfast ? 64 : 128;
  return true;
}


// ---- TMA-reduce epilogue (fused ABC) ------------------------------------------
// C target views as tensor-map boxes of 32 tile rows x 128 tile columns, dims
// (column low 16, column high..., rows...), 128-byte swizzle: the smem piece is
// [row][column / 16][column % 16].  Needs the C tensor's unit-stride label to
// lead the J bundle's tile order.  x part = rows (I), k part = columns (J).
constexpr int kRedRows = 16;

bool plan_cred_side(const stc_bundle &rb, const Tiling &tr, const stc_bundle &cb, const Tiling &tc, int level,
                    const double *data, int64_t base, TmaSide &ts) {
  if (tr.nbox == 0 || tc.nbox == 0) return false;
  const int64_t Q = (int64_t)1 << level;
  if ((bundle_len(rb) / Q) % BM != 0 || (bundle_len(cb) / Q) % BN != 0) return false;
  int64_t tbr[STC_MAX_LABELS], tbc[STC_MAX_LABELS];
  int orr[STC_MAX_LABELS], oc[STC_MAX_LABELS], nor = 0, noc = 0;
  if (!tile_subbox(rb, tr, kRedRows, tbr, orr, nor) || !tile_subbox(cb, tc, BN, tbc, oc, noc)) return false;
  struct Dim {
    int64_t ext, str, box;
    bool isx;
  };
  std::vector<Dim> dims;
  if (noc == 0 || cb.str[oc[0]] != 1) return false;
  const int64_t e0 = cb.ext[oc[0]], b0 = tbc[oc[0]];
  // the unit-stride label's tile extent: 16+ doubles -> 128-byte rows (128B swizzle);
  // exactly 8 (a quadrant split of that label, e.g. cfg5's k at L2) -> 64-byte rows
  // (64B swizzle; GemmArgs::cred8)
  const bool w8 = b0 == 8;
  if (w8) {
    dims.push_back({e0, 1, 8, false});
  } else {
    if (b0 < 16 || b0 % 16 != 0 || (b0 > 16 && e0 % 16 != 0)) return false;
    dims.push_back({b0 > 16 ? 16 : e0, 1, 16, false});
    if (b0 > 16) dims.push_back({e0 / 16, 16, b0 / 16, false});
  }
  for (int j = 1; j < noc; ++j) dims.push_back({cb.ext[oc[j]], cb.str[oc[j]], tbc[oc[j]], false});
  for (int j = 0; j < nor; ++j) dims.push_back({rb.ext[orr[j]], rb.str[orr[j]], tbr[orr[j]], true});
  for (int pass = 0; pass < 2; ++pass) {
    const stc_bundle &b = pass == 0 ? rb : cb;
    const int64_t *tb = pass == 0 ? tbr : tbc;
    for (int d = 0; d < b.nlab; ++d)
      if (b.ext[d] > 1 && tb[d] == 1) dims.push_back({b.ext[d], b.str[d], 1, pass == 0});
  }
  merge_dims(dims);
  if (dims.size() > 5) return false;
  for (size_t d = 0; d < dims.size(); ++d) {
    if (dims[d].str <= 0 || dims[d].box > 256 || dims[d].ext >= (int64_t)1 << 31) return false;
    if (d > 0 && ((dims[d].str % 2) != 0 || dims[d].str * 8 >= ((int64_t)1 << 40))) return false;
  }
  if ((reinterpret_cast<uintptr_t>(data + base) & 15) != 0) return false;
  for (int part = 0; part < 2; ++part) {
    std::vector<int> idx;
    for (size_t d = 0; d < dims.size(); ++d)
      if (dims[d].isx == (part == 0)) idx.push_back((int)d);
    if (idx.empty() || idx.size() > 4) return false;
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return dims[a].str > dims[b].str; });
    for (size_t i = 0; i + 1 < idx.size(); ++i)
      if (dims[idx[i]].str < dims[idx[i + 1]].str * dims[idx[i + 1]].ext) return false;
    ts.np[part] = (int)idx.size();
    for (size_t i = 0; i < idx.size(); ++i) {
      ts.pstr[part][i] = dims[idx[i]].str;
      ts.src[idx[i]] = part * 4 + (int)i;
    }
    for (size_t i = idx.size(); i < 4; ++i) ts.pstr[part][i] = 1;
  }
  ts.rank = (int)dims.size();
  for (int d = 0; d < ts.rank; ++d) {
    ts.dims[d] = (cuuint64_t)dims[d].ext;
    ts.box[d] = (cuuint32_t)dims[d].box;
    if (d > 0) ts.strides[d - 1] = (cuuint64_t)(dims[d].str * 8);
  }
  for (int d = ts.rank; d < 5; ++d) ts.src[d] = 0;
  ts.swizzle = w8 ? 64 : 128;
  return true;
}

// C quadrant tiles are boxes the TMA-reduce epilogue can address (alignment of
// the actual pointer aside): the fused kernel's ABC C updates stay off the SMs.
bool c_boxes_regular(const stc_problem *p, const Tiling &ti, const Tiling &tj, int level) {
  TmaSide sc;
  return plan_cred_side(p->c_row, ti, p->c_col, tj, level, nullptr, p->c_base, sc);
}

FusedSides direct_sides(const stc_problem *p, const Plan &pl) {
  FusedSides f;
  f.ax = p->a_row;
  f.ak = p->a_col;
  f.bk = p->b_row;
  f.bx = p->b_col;
  f.tax = pl.ti;
  f.tak = pl.tp;
  f.tbk = pl.tp;
  f.tbx = pl.tj;
  f.akf = pl.a_kfast;
  f.bkf = pl.b_kfast;
  f.a_base = p->a_base;
  f.b_base = p->b_base;
  const int64_t st[4] = {pl.ar, pl.ac, pl.br, pl.bc};
  const int64_t ln[4] = {pl.Q * pl.mq_pad, pl.Q * pl.kq_pad, pl.Q * pl.kq_pad, pl.Q * pl.nq_pad};
  const int64_t vb[4] = {0, p->a_base, 0, p->b_base};  // build_plan: ac carries a_base, bc carries b_base
  for (int i = 0; i < 4; ++i) {
    f.start[i] = st[i];
    f.len[i] = ln[i];
    f.vbase[i] = vb[i];
  }
  f.qxa = bundle_len(p->a_row) / pl.Q;
  f.qk = bundle_len(p->a_col) / pl.Q;
  f.qxb = bundle_len(p->b_col) / pl.Q;
  return f;
}

// Repacked sides: quadrant block (r, c) of A is a dense mq_pad x kq_pad block
// [k][x] (unit stride in x) or [x][k] (unit stride in k, like the source), block
// index r * Q + c; B's block (r, c) (P quadrant r, J quadrant c) likewise with
// nq_pad.  Expressed as two-label bundles (x | quadrant, k | quadrant) so the
// fused planner treats them like any other tensor.
void packed_bundle(stc_bundle &b, int64_t len, int64_t stride, int64_t Q, int64_t qstride) {
  memset(&b, 0, sizeof(b));
  b.nlab = Q > 1 ? 2 : 1;
  b.ext[0] = len;
  b.str[0] = stride;
  if (Q > 1) {
    b.ext[1] = Q;
    b.str[1] = qstride;
  }
}

FusedSides packed_sides(const Plan &pl) {
  FusedSides f;
  const int64_t Q = pl.Q, mq = pl.mq_pad, nq = pl.nq_pad, kq = pl.kq_pad;
  const int64_t blkA = mq * kq, blkB = nq * kq;
  f.akf = pl.a_kfast;
  f.bkf = pl.b_kfast;
  // A: x quadrant r (block row), k quadrant c (block column)
  packed_bundle(f.ax, mq, f.akf ? kq : 1, Q, Q * blkA);
  packed_bundle(f.ak, kq, f.akf ? 1 : mq, Q, blkA);
  // B: k quadrant r (block row), x quadrant c (block column)
  packed_bundle(f.bk, kq, f.bkf ? 1 : nq, Q, Q * blkB);
  packed_bundle(f.bx, nq, f.bkf ? kq : 1, Q, blkB);
  const int64_t keyx[2] = {1, 2}, keyk[2] = {1, 2};  // tile order: the block dims in natural order
  f.tax = make_tiling(f.ax, pl.level, keyx, false);
  f.tak = make_tiling(f.ak, pl.level, keyk, false);
  f.tbk = make_tiling(f.bk, pl.level, keyk, false);
  f.tbx = make_tiling(f.bx, pl.level, keyx, false);
  const int64_t st[4] = {pl.ar, pl.ac, pl.br, pl.bc};
  const int64_t ln[4] = {Q * mq, Q * kq, Q * kq, Q * nq};
  for (int i = 0; i < 4; ++i) {
    f.start[i] = st[i];
    f.len[i] = ln[i];
    f.vbase[i] = 0;
  }
  f.qxa = mq;
  f.qk = kq;
  f.qxb = nq;
  return f;
}

// Naive: the packed operand sums of each term slot ([k][x] or [x][k] blocks,
// slot stride pa_slot / pb_slot) as bundles (x | slot, k); the slot x vectors
// dxa / dxb are per-slot (mode 2), so a term's view is its own slot block.
FusedSides naive_sides(const Plan &pl) {
  FusedSides f;
  const int64_t mq = pl.mq_pad, nq = pl.nq_pad, kq = pl.kq_pad, nb = pl.batch;
  f.akf = pl.a_kfast;
  f.bkf = pl.b_kfast;
  packed_bundle(f.ax, mq, f.akf ? kq : 1, nb, pl.pa_slot);
  packed_bundle(f.ak, kq, f.akf ? 1 : mq, 1, 0);
  packed_bundle(f.bk, kq, f.bkf ? 1 : nq, 1, 0);
  packed_bundle(f.bx, nq, f.bkf ? kq : 1, nb, pl.pb_slot);
  auto natural = [](int64_t len) {
    Tiling t;
    t.nbox = 1;
    t.box_ext[0] = len;
    t.order[0] = 0;
    return t;
  };
  f.tax = natural(mq);
  f.tak = natural(kq);
  f.tbk = natural(kq);
  f.tbx = natural(nq);
  const int64_t st[4] = {pl.dxa, pl.dka, pl.dkb, pl.dxb};
  const int64_t ln[4] = {nb * mq, kq, kq, nb * nq};
  for (int i = 0; i < 4; ++i) {
    f.start[i] = st[i];
    f.len[i] = ln[i];
    f.vbase[i] = 0;
  }
  f.qxa = mq;
  f.qk = kq;
  f.qxb = nq;
  return f;
}

// Pre-summed sides from their slots (naive_sides), the others' own views (direct_sides).
FusedSides mixed_sides(const stc_problem *p, const Plan &pl) {
  const FusedSides n = naive_sides(pl);
  if (pl.presum_sides == 3 || pl.variant == STC_VARIANT_NAIVE) return n;
  FusedSides f = direct_sides(p, pl);
  if (pl.presum_sides & 1) {
    f.ax = n.ax;
    f.ak = n.ak;
    f.tax = n.tax;
    f.tak = n.tak;
    f.akf = n.akf;
    f.a_base = n.a_base;
    f.qxa = n.qxa;
    for (int i = 0; i < 2; ++i) {
      f.start[i] = n.start[i];
      f.len[i] = n.len[i];
      f.vbase[i] = n.vbase[i];
    }
  }
  if (pl.presum_sides & 2) {
    f.bx = n.bx;
    f.bk = n.bk;
    f.tbx = n.tbx;
    f.tbk = n.tbk;
    f.bkf = n.bkf;
    f.b_base = n.b_base;
    f.qxb = n.qxb;
    for (int i = 2; i < 4; ++i) {
      f.start[i] = n.start[i];
      f.len[i] = n.len[i];
      f.vbase[i] = n.vbase[i];
    }
  }
  return f;
}

// The packed sides' pool vectors (mode 2), written over ar, ac, br, bc once the
// operands are packed (the ops tables then address the packed blocks unchanged).
void packed_vecs(const Plan &pl, const FusedSides &f, VecDesc out[4]) {
  const stc_bundle *b[4] = {&f.ax, &f.ak, &f.bk, &f.bx};
  for (int i = 0; i < 4; ++i) {
    VecDesc &d = out[i];
    memset(&d, 0, sizeof(d));
    d.mode = 2;
    d.out_start = f.start[i];
    d.nq = pl.Q;
    d.q_len = d.q_len_pad = d.len = b[i]->ext[0];
    d.stride = b[i]->str[0];
    d.base = pl.Q > 1 ? b[i]->str[1] : 0;
  }
}

// Fused-kernel plan for ABC / AB (terms of at most 8 views per chunk: L <= 2):
// tensor maps, the coordinate-table jobs and the kernel arguments.
// STC_FUSED=0 disables.  A / B null: layout check only (no maps).
bool plan_fused(const stc_problem *p, const Plan &pl, const FusedSides &fs, const double *A, const double *B,
                const double *C, GemmArgs &g, CUtensorMap maps[3], CoordJobs &jobs) {
  if (const char *e = stc_env("STC_FUSED"))
    if (atoi(e) == 0) return false;
  if (pl.flags & (STC_FLAG_FORCE_SLOW | STC_FLAG_REFERENCE_TILING)) return false;
  // Naive and pre-summed sides: one packed view per side
  const bool all_slots = pl.variant == STC_VARIANT_NAIVE || (pl.presum && pl.presum_sides == 3);
  const int va = all_slots || (pl.presum && (pl.presum_sides & 1)) ? 1 : pl.max_ops;
  const int vb = all_slots || (pl.presum && (pl.presum_sides & 2)) ? 1 : pl.max_ops;
  const int umax = va + vb;
  const size_t sd = fused_stage_doubles2(va, vb, pl.tshape);
  const int S = fused_stages(sd);
  if (umax > 8 || S < 2) return false;
  TmaSide sa, sb;
  if (!plan_fused_side(fs.ax, fs.tax, fs.ak, fs.tak, fs.qxa, fs.qk, fs.akf, A, fs.a_base, sa, pl.tm)) return false;
  if (!plan_fused_side(fs.bx, fs.tbx, fs.bk, fs.tbk, fs.qxb, fs.qk, fs.bkf, B, fs.b_base, sb, pl.tn)) return false;
  if (!A || !B) return true;
  if (!encode_side(sa, A, fs.a_base, maps[0]) || !encode_side(sb, B, fs.b_base, maps[1])) return false;
  const TmaSide *ss[2] = {&sa, &sb};
  for (int sd = 0; sd < 2; ++sd) {
    g.tm_rank[sd] = ss[sd]->rank;
    for (int d = 0; d < 5; ++d) g.tm_src[sd][d] = ss[sd]->src[d];
    for (int part = 0; part < 2; ++part) {
      g.tm_np[sd][part] = ss[sd]->np[part];
      for (int i = 0; i < 4; ++i) g.tm_pstr[sd][part][i] = ss[sd]->pstr[part][i];
    }
  }
  // pool vectors ar (A x), ac (A k), br (B k), bc (B x)
  const int vsd[4] = {0, 0, 1, 1}, vpart[4] = {0, 1, 1, 0};
  jobs.n = 4;
  for (int j = 0; j < 4; ++j) {
    CoordJob &jb = jobs.job[j];
    jb.start = fs.start[j];
    jb.count = fs.len[j] / 8;
    jb.base = fs.vbase[j];
    jb.np = ss[vsd[j]]->np[vpart[j]];
    for (int i = 0; i < 4; ++i) jb.str[i] = ss[vsd[j]]->pstr[vpart[j]][i];
  }
  g.a_kfast = fs.akf;
  g.b_kfast = fs.bkf;
  // ABC: C updates by TMA reduce-add when the C targets are regular boxes (STC_CRED=0 disables)
  g.cred = 0;
  TmaSide sc;
  if (pl.variant == STC_VARIANT_ABC && C && !(stc_env("STC_CRED") && atoi(stc_env("STC_CRED")) == 0) &&
      fused_stages_red(sd) >= 2 &&
      plan_cred_side(p->c_row, pl.ti, p->c_col, pl.tj, pl.level, C, p->c_base, sc) &&
      encode_side(sc, C, p->c_base, maps[2])) {
    g.cred = 1;
    g.cred8 = sc.swizzle == 64;
    g.tm_rank[2] = sc.rank;
    for (int d = 0; d < 5; ++d) g.tm_src[2][d] = sc.src[d];
    for (int part = 0; part < 2; ++part) {
      g.tm_np[2][part] = sc.np[part];
      for (int i = 0; i < 4; ++i) g.tm_pstr[2][part][i] = sc.pstr[part][i];
    }
    // pool vectors cr (rows, base 0) and cc (columns, base c_base)
    const int64_t lens[2] = {pl.Q * rup(cdiv(bundle_len(p->c_row), pl.Q), BM), pl.Q * rup(cdiv(bundle_len(p->c_col), pl.Q), BN)};
    const int64_t starts[2] = {pl.cr, pl.cc}, bases[2] = {0, p->c_base};
    for (int part = 0; part < 2; ++part) {
      CoordJob &jb = jobs.job[jobs.n++];
      jb.start = starts[part];
      jb.count = lens[part] / 8;
      jb.base = bases[part];
      jb.np = sc.np[part];
      for (int i = 0; i < 4; ++i) jb.str[i] = sc.pstr[part][i];
    }
  }
  g.tma = 0;
  g.umax = umax;
  g.one_view = umax == 2;  // L0, Naive slots, pre-summed slots: one view per side, sign +1
  g.stages = g.cred ? fused_stages_red(sd) : S;
  if (pl.stage_cap >= 2) g.stages = std::min(g.stages, pl.stage_cap);  // stc_problem.tiling
  g.stage_dbl = (int32_t)sd;
  g.tshape = pl.tshape;
  // summing warpgroup when some side has more than one view per chunk (L >= 1):
  // STC_PRESUM = 0 (the consumers form every sum), 1 (A side; default), 3 (both sides)
  // (3 with one-sided A slots -- the summers form the 256-wide B sums -- measured slower:
  // cfg3 2^24 N_a = 16 L2 4.35 vs 4.01 ms)
  g.psum = 0;
  if (umax > 2) {
    const char *e = stc_env("STC_PRESUM");
    g.psum = e ? atoi(e) & 3 : 1;
    if (g.psum == 2) g.psum = 3;
  }
  g.kchunks = (int)(pl.kq_pad / kFusedK);
  return true;
}

// k_presum arguments for one side (0: A, 1: B) of the exec-order terms [t0, t1).
PresumArgs presum_args(const Plan &pl, int side, const double *D, double *out, const int64_t *pool, int t0, int t1) {
  PresumArgs a{};
  a.D = D;
  a.pool = pool;
  a.out = out;
  a.level = pl.level;
  a.side = side;
  for (int t = 0; t <= kPresumMaxTerms; ++t) a.slot[t] = -1;
  for (int t = t0; t < t1; ++t) a.slot[pl.seq[t]] = (int16_t)(t - t0);
  a.klen = pl.kq_pad;
  if (side == 0) {
    a.slot_stride = pl.pa_slot;
    a.xv = pl.ar;
    a.kv = pl.ac;
    a.xlen = pl.mq_pad;
    a.kfast = pl.a_kfast;
    a.ustep = pl.a_ustep;
    a.ugroup = pl.a_ugroup;
  } else {
    a.slot_stride = pl.pb_slot;
    a.xv = pl.bc;
    a.kv = pl.br;
    a.xlen = pl.nq_pad;
    a.kfast = pl.b_kfast;
    a.ustep = pl.b_ustep;
    a.ugroup = pl.b_ugroup;
  }
  return a;
}

// Plans depend only on the problem descriptor, the grid size and the STC_*
// planning knobs; repeated calls on one problem (benchmark loops, the pieces of
// stc_contract_host) reuse them instead of re-planning (~0.1 ms each).
struct PlanEntry {
  stc_problem prob;
  int grid;
  std::string env;
  std::shared_ptr<const Plan> plan;  // shared with the calls using it (no per-call copy)
};
std::mutex g_plan_mu;
std::vector<PlanEntry> g_plans;
size_t g_plan_next = 0;
constexpr size_t kPlanCache = 128;  // (a 4 x 8 host grid alone plans 32-34 pieces)

std::string plan_env() {
  static const char *knobs[] = {"STC_WORKSPACE_CAP_MB", "STC_EXEC_ORDER", "STC_PACK", "STC_TMA_PROMO",
                                "STC_TMA", "STC_TMA_PF", "STC_FUSED", "STC_CRED", "STC_PRESUM",
                                "STC_ABC_DENSE", "STC_TSHAPE", "STC_PRESUM_OPS", "STC_NO_USTEP", "STC_EPI_OFFLOAD", "STC_TERM_INNER",
                                "STC_PRESUM_SIDES"};
  std::string key;
  for (const char *k : knobs) {
    const char *v = stc_env(k);
    key += v ? v : "\x01";
    key += '\0';
  }
  return key;
}

int cached_plan(const stc_problem *p, std::shared_ptr<const Plan> &out, int grid_hint) {
  if (!p) return fail(STC_EINVAL, "null problem");
  env_refresh();
  const std::string env = plan_env();
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    for (const PlanEntry &e : g_plans)
      if (e.grid == grid_hint && e.env == env && memcmp(&e.prob, p, sizeof(stc_problem)) == 0) {
        out = e.plan;
        return STC_OK;
      }
  }
  auto pl = std::make_shared<Plan>();
  if (int rc = build_plan(p, *pl, grid_hint)) return rc;
  out = pl;
  std::lock_guard<std::mutex> lk(g_plan_mu);
  PlanEntry e{*p, grid_hint, env, out};
  if (g_plans.size() < kPlanCache) {
    g_plans.push_back(std::move(e));
  } else {
    g_plans[g_plan_next] = std::move(e);
    g_plan_next = (g_plan_next + 1) % kPlanCache;
  }
  return STC_OK;
}

}  // namespace

namespace stc {
int set_error(int code, const char *msg) {
  g_err = msg;
  return code;
}

// Whether stc_contract runs the problem ticketed (ABC, C updated by the kernel)
// rather than through dense M slots and an accumulate kernel (stc_host.cu).
bool plan_ticketed(const stc_problem *p) {
  std::shared_ptr<const Plan> pl;
  const int sms = gemm_max_grid(MAX_OPS);
  if (cached_plan(p, pl, sms > 0 ? sms : 0)) return false;
  return pl->ticketed;
}

bool plan_slot_bytes(const stc_problem *p, size_t &a_bytes, size_t &b_bytes) {
  a_bytes = b_bytes = 0;
  std::shared_ptr<const Plan> pl;
  const int sms = gemm_max_grid(MAX_OPS);
  if (cached_plan(p, pl, sms > 0 ? sms : 0)) return false;
  if (!pl->presum || pl->presum_sides != 3 || pl->nbatches != 1 || pl->variant == STC_VARIANT_NAIVE) return false;
  a_bytes = (size_t)pl->batch * pl->pa_slot * 8;
  b_bytes = (size_t)pl->batch * pl->pb_slot * 8;
  return true;
}

void set_slot_override(const SlotOverride *o) {
  g_slot_ovr_set = o != nullptr;
  g_slot_ovr = o ? *o : SlotOverride{};
}

}  // namespace stc

// ======================================================================== ABI
extern "C" {

const char *stc_last_error(void) { return g_err.c_str(); }
int stc_abi_version(void) { return STC_ABI_VERSION; }

int stc_set_kernel_events(void *before, void *after) {
  g_ev_before = reinterpret_cast<cudaEvent_t>(before);
  g_ev_after = reinterpret_cast<cudaEvent_t>(after);
  return STC_OK;
}

int stc_set_c_ready(const int32_t *c_ready) {
  g_c_ready = c_ready;
  return STC_OK;
}

int stc_workspace_size(const stc_problem *p, size_t *bytes) {
  std::shared_ptr<const Plan> pl;
  const int sms = gemm_max_grid(MAX_OPS);  // per-CTA scratch is sized by the launch grid (0 without a device)
  if (int rc = cached_plan(p, pl, sms > 0 ? sms : 0)) return rc;
  if (bytes) *bytes = pl->total;
  return STC_OK;
}

// The launch sequence of one contraction on stream s (stc_contract: checks, operand
// mode, snapshot and graph handling).  `snap`: the plan's snapshot of the constant
// workspace region for this operand mode, already ordered before s (null: build it).
static int contract_run(const stc_problem *p, const Plan &pl, const double *A, const double *B, double *C, char *ws,
                 cudaStream_t s, const int32_t *c_ready, cudaEvent_t ev_before, cudaEvent_t ev_after, bool direct,
                 bool packed, int mode, int dev, const void *snap, const SlotOverride *ovr, stc_stats *stats) {
  // The constant region is read where it lives: in the plan's snapshot once there is
  // one (nothing to restore), else in the workspace, where this call builds it.  Only
  // the tickets and work counters at its end are per call (zeroed in the workspace).
  char *cw = snap ? const_cast<char *>(static_cast<const char *>(snap)) : ws;
  int64_t *pool = reinterpret_cast<int64_t *>(cw + pl.off_pool);
  int64_t *pool2 = reinterpret_cast<int64_t *>(cw + pl.off_pool2);  // the original vectors (repacking)
  int64_t *kbs = reinterpret_cast<int64_t *>(cw + pl.off_kbs);
  int32_t *tickets = reinterpret_cast<int32_t *>(ws + pl.off_tickets);
  int32_t *counters = reinterpret_cast<int32_t *>(ws + pl.off_counters);
  int4 *coords = reinterpret_cast<int4 *>(cw + pl.off_coords);
  int64_t launches = 0;
  bool tma = false;  // operand units staged by tensor-map box loads
  stc_stats st{};
  g_stage_launches = 0;
  const int tiles_m = (int)(pl.mq_pad / pl.tm), tiles_n = (int)(pl.nq_pad / pl.tn);
  const int64_t P = (int64_t)tiles_m * tiles_n;
  const int T = (int)pl.terms.size();
  const bool slots = pl.variant == STC_VARIANT_NAIVE || pl.presum;
  Resident *res = pl.res.get();
  const bool restored = snap != nullptr;
  // per call: zero the tickets and counters (by the first k_presum launch when there is one)
  int32_t *const zero = restored ? tickets : nullptr;
  const int64_t zero_words = (int64_t)((pl.off_const - pl.off_tickets) / 4);
  const bool shared_slots = ovr && pl.presum && pl.presum_sides == 3 && pl.nbatches == 1;
  const bool skip_a = shared_slots && ovr->skip_a, skip_b = shared_slots && ovr->skip_b;
  const bool presum_runs = pl.presum && !(skip_a && skip_b);
  if (restored && !presum_runs) {
    CU(cudaMemsetAsync(ws + pl.off_tickets, 0, pl.off_const - pl.off_tickets, s), "zero tickets");
  } else if (!restored) {
    if (int rc = upload(pl.vecs.data(), pl.vecs.size() * sizeof(VecDesc), ws + pl.off_vecs, s, ws + pl.off_tickets,
                        pl.off_const - pl.off_tickets))
      return rc;
    CU(launch_build_pool(reinterpret_cast<VecDesc *>(ws + pl.off_vecs), (int)pl.vecs.size(), pl.pool_len, pool, s),
       "k_build_pool");
    CU(launch_chunk_strides(pool, pl.pool_len / BK, kbs, s), "k_chunk_strides");
    launches += 2;
    if (packed) {  // a copy of the original vectors for k_pack_views (pool gets the packed ones)
      CU(launch_build_pool(reinterpret_cast<VecDesc *>(ws + pl.off_vecs), (int)pl.vecs.size(), pl.pool_len, pool2, s),
         "k_build_pool(2)");
      ++launches;
    }
  }
  auto save_snapshot = [&]() -> int {
    if (restored || !res) return STC_OK;
    CU(res->save(mode, dev, ws, pl.off_const, s), "snapshot");
    return STC_OK;
  };

  // Fused kernel set-up on the operands' own views or their repacked blocks: the
  // repacking runs every call (it reads A and B), the rest is constant.
  // (errors are returned negated: 0 = the gather kernel, 1 = fused kernel prepared)
#define CUN(expr, what)                                  \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return -cuda_fail(_e, what);  \
  } while (0)
  auto prepare_fused = [&](GemmArgs &gf, CUtensorMap *maps, const double *Cp) -> int {
    CoordJobs jobs{};
    if (packed) {
      double *PA = reinterpret_cast<double *>(ws + pl.off_pka);
      double *PB = reinterpret_cast<double *>(ws + pl.off_pkb);
      PackArgs pa{pl.ar, pl.ac, pl.mq_pad, pl.kq_pad, (int32_t)pl.Q, 1, pl.a_kfast, 0, pl.a_ustep, pl.a_ugroup, 0};
      PackArgs pb{pl.bc, pl.br, pl.nq_pad, pl.kq_pad, (int32_t)pl.Q, 0, pl.b_kfast, 0, pl.b_ustep, pl.b_ugroup, 0};
      CUN(launch_pack_views(A, pool2, pa, PA, s), "k_pack_views(A)");
      CUN(launch_pack_views(B, pool2, pb, PB, s), "k_pack_views(B)");
      launches += 2;
      const FusedSides fs = packed_sides(pl);
      if (!restored) {
        VecDesc pv[4];
        packed_vecs(pl, fs, pv);
        VecDesc *d_pv = reinterpret_cast<VecDesc *>(ws + pl.off_vecs) + pl.vecs.size();
        if (int rc = upload(pv, sizeof(pv), d_pv, s)) return -rc;
        CUN(launch_build_pool(d_pv, 4, pl.pool_len, pool, s), "k_build_pool(packed)");
        ++launches;
      }
      if (!plan_fused(p, pl, fs, PA, PB, Cp, gf, maps, jobs)) return -fail(STC_EINVAL, "internal: packed plan");
      gf.A = PA;
      gf.B = PB;
    } else if (direct) {
      if (!plan_fused(p, pl, direct_sides(p, pl), A, B, Cp, gf, maps, jobs))
        return -fail(STC_EINVAL, "internal: direct plan");
      gf.A = A;
      gf.B = B;
    } else {
      return 0;  // the gather kernel
    }
    gf.coords = coords;
    if (!restored) {
      CUN(launch_pool_coords(pool, coords, jobs, s), "k_pool_coords");
      ++launches;
    }
    return 1;
  };
#undef CUN

  GemmArgs g{};
  g.pool = pool;
  g.c_ready = c_ready;
  g.tiles_m = tiles_m;
  g.tiles_n = tiles_n;
  g.rows_valid = (int32_t)pl.mq;
  g.cols_valid = (int32_t)pl.nq;
  // row-padding warp tiles (the last row tile at most half valid) but no column ones
  g.warp_map = (pl.mq % BM != 0 && pl.mq % BM <= 64) && !(pl.nq % BN != 0 && pl.nq % BN <= 96);
  g.kchunks = (int)(pl.kq_pad / BK);
  g.group_m = 8;
  if (const char *e = stc_env("STC_GROUP_M")) g.group_m = std::max(1, atoi(e));
  g.term_inner = pl.term_inner ? 1 : 0;
  g.max_ops = pl.max_ops;
  g.nraw = gemm_nraw(pl.max_ops);
  g.kwin = gemm_kwin(pl.max_ops);
  g.kbs = kbs;
  g.force_slow = (pl.flags & STC_FLAG_FORCE_SLOW) ? 1 : 0;
  g.tickets = tickets;

  if (pl.ticketed) {
    char *tab = cw + pl.off_tab;
    std::vector<char> host(pl.tab_bytes);
    size_t o = 0;
    memcpy(host.data() + o, pl.tdesc.data(), pl.tdesc.size() * sizeof(TermDesc));
    g.terms = reinterpret_cast<const TermDesc *>(tab + o);
    o += pl.tdesc.size() * sizeof(TermDesc);
    memcpy(host.data() + o, pl.ops.data(), pl.ops.size() * sizeof(OpDesc));
    g.ops = reinterpret_cast<const OpDesc *>(tab + o);
    o += pl.ops.size() * sizeof(OpDesc);
    memcpy(host.data() + o, pl.tgts.data(), pl.tgts.size() * sizeof(TgtDesc));
    g.tgts = reinterpret_cast<const TgtDesc *>(tab + o);
    if (!restored)
      if (int rc = upload(host.data(), host.size(), tab, s)) return rc;
    g.A = A;
    g.B = B;
    g.C = C;
    g.nterms = T;
    g.total_items = (int)(P * T);
    g.a_kfast = pl.a_kfast;
    g.b_kfast = pl.b_kfast;
    g.dense_out = 0;
    g.use_tickets = T > 1;
    g.counter = counters;
    const int grid = (int)std::min<int64_t>(pl.grid, g.total_items);
    CUtensorMap maps[3];
    GemmArgs gf = g;
    if (pl.presum) {
      // pre-summed operands: per batch of terms (exec order), one k_presum pass per side
      // writes the batch's operand sums into their slots, then one fused launch runs
      // the batch's items with one view per side (C updates ticket-ordered as ever)
      double *PA = shared_slots && ovr->pa ? ovr->pa : reinterpret_cast<double *>(ws + pl.off_pa);
      double *PB = shared_slots && ovr->pb ? ovr->pb : reinterpret_cast<double *>(ws + pl.off_pb);
      CoordJobs jobs{};
      if (!plan_fused(p, pl, naive_sides(pl), PA, PB, C, gf, maps, jobs))
        return fail(STC_EINVAL, "internal: pre-summed plan");
      gf.A = PA;
      gf.B = PB;
      gf.coords = coords;
      if (!restored) {
        CU(launch_pool_coords(pool, coords, jobs, s), "k_pool_coords");
        ++launches;
      }
      if (int rc = save_snapshot()) return rc;
      if (gf.cred) gf.mscratch = reinterpret_cast<double *>(ws + pl.off_mscr);
      for (int bi = 0; bi < pl.nbatches; ++bi) {
        const int t0 = bi * pl.batch, nb = std::min(T - t0, pl.batch);
        if (presum_runs) {
          PresumArgs pa = presum_args(pl, 0, A, skip_a ? nullptr : PA, pool, t0, t0 + nb);
          if (bi == 0 && zero) {
            pa.zero = zero;
            pa.zero_words = zero_words;
          }
          CU(launch_presum2(pa, presum_args(pl, 1, B, skip_b ? nullptr : PB, pool, t0, t0 + nb), s), "k_presum");
        }
        if (shared_slots && ovr->after_presum) CU(cudaEventRecord(ovr->after_presum, s), "cudaEventRecord");
        gf.terms = g.terms + t0;
        gf.nterms = nb;
        gf.total_items = (int)(P * nb);
        gf.counter = counters + bi;
        if (ev_before && bi == 0) CU(cudaEventRecord(ev_before, s), "cudaEventRecord");
        CU(launch_fused(gf, (int)std::min<int64_t>(pl.grid, gf.total_items), s, maps), "k_strassen_fused");
        launches += 2;
      }
      if (ev_after) CU(cudaEventRecord(ev_after, s), "cudaEventRecord");
      tma = true;
      st.fast_updates = gf.cred ? (int64_t)P * (int64_t)pl.tgts.size() : 0;
      st.slow_updates = gf.cred ? 0 : (int64_t)P * (int64_t)pl.tgts.size();
    } else {
      const int fz = prepare_fused(gf, maps, C);
      if (fz < 0) return -fz;
      if (!fz) tma = plan_tma(p, pl, A, B, g, maps);  // the gather kernel (host set-up only)
      if (int rc = save_snapshot()) return rc;
      if (fz) {
        // fused kernel: TMA boxes of 128 x 8.  C updates by the producer warpgroup's three
        // spare warps from dense M tiles with the TMA reduce-add epilogue (no FP64 work in
        // those warps); without TMA reduce (C not box-regular: only L0 reaches here) the
        // consumers' own load/add/store epilogue (the spare warps' DADDs starve behind the
        // DMMAs); STC_EPI_OFFLOAD overrides, 8-wide C boxes always go to the spare warps
        tma = !packed;
        const char *eo = stc_env("STC_EPI_OFFLOAD");
        const int offload = (eo ? atoi(eo) : (gf.cred ? 1 : 0)) || (gf.cred && gf.cred8);
        if (offload) gf.mscratch = reinterpret_cast<double *>(ws + pl.off_mscr);
        if (ev_before) CU(cudaEventRecord(ev_before, s), "cudaEventRecord");
        CU(launch_fused(gf, grid, s, maps), "k_strassen_fused");
      } else {
        if (ev_before) CU(cudaEventRecord(ev_before, s), "cudaEventRecord");
        CU(launch_gemm(g, grid, s, tma ? maps : nullptr), "k_strassen_gemm");
      }
      if (ev_after) CU(cudaEventRecord(ev_after, s), "cudaEventRecord");
      ++launches;
      // C-tile updates: by TMA reduce-add boxes (the reference's fast store_tile path,
      // _jit.py:166-176) or by the load/add/store scatter epilogue (its slow path)
      const int64_t upd = (int64_t)P * (int64_t)pl.tgts.size();
      st.fast_updates = (fz && gf.cred) ? upd : 0;
      st.slow_updates = (fz && gf.cred) ? 0 : upd;
    }
  } else {
    // dense M: per-term operand slots (Naive's explicit copies, pre-summed ABC / AB
    // operands) or the operands' own / repacked views (AB); per batch of terms the slots,
    // one DMMA launch writing dense M, one ordered accumulate into C
    double *M = reinterpret_cast<double *>(ws + pl.off_M);
    double *PA = shared_slots && ovr->pa ? ovr->pa : reinterpret_cast<double *>(ws + pl.off_pa);
    double *PB = shared_slots && ovr->pb ? ovr->pb : reinterpret_cast<double *>(ws + pl.off_pb);
    const bool slot_a = slots && (pl.variant == STC_VARIANT_NAIVE || (pl.presum_sides & 1));
    const bool slot_b = slots && (pl.variant == STC_VARIANT_NAIVE || (pl.presum_sides & 2));
    struct Batch {
      int t0, t1;
      const TermDesc *d_g, *d_ua, *d_ub;
      const OpDesc *d_ops;
      AccArgs aa;
      int64_t nupd;
    };
    std::vector<Batch> batches;
    // pass 1: the batches' tables (constant: uploaded unless restored)
    for (int bi = 0; bi < pl.nbatches; ++bi) {
      const int t0 = bi * pl.batch, t1 = std::min(T, t0 + pl.batch);
      const int nb = t1 - t0;
      std::vector<TermDesc> gterms(nb), uA(nb), uB(nb);
      std::vector<OpDesc> ops;
      for (int t = t0; t < t1; ++t) {
        const Term &tm = pl.terms[pl.seq[t]];
        const int slot = t - t0;
        TermDesc ua{}, ub{}, gd{};
        ua.a_first = (int)ops.size();
        ua.a_count = (int)tm.a.size();
        for (const Op &op : tm.a) {
          int64_t r, c;
          quad_rc(op.q, pl.level, r, c);
          ops.push_back({pl.ar + r * pl.mq_pad, pl.ac + c * pl.kq_pad, 0, (double)op.s});
        }
        ub.a_first = (int)ops.size();
        ub.a_count = (int)tm.b.size();
        for (const Op &op : tm.b) {
          int64_t r, c;
          quad_rc(op.q, pl.level, r, c);
          ops.push_back({pl.bc + c * pl.nq_pad, pl.br + r * pl.kq_pad, 0, (double)op.s});
        }
        ua.m_slot = ub.m_slot = gd.m_slot = slot;
        if (slots) {  // a pre-summed side: the term's slot; the other (one-sided): its own views
          gd.a_first = ua.a_first;
          gd.a_count = ua.a_count;
          gd.b_first = ub.a_first;
          gd.b_count = ub.a_count;
          if (slot_a) {
            gd.a_first = (int)ops.size();
            gd.a_count = 1;
            ops.push_back({pl.dxa + slot * pl.mq_pad, pl.dka, 0, 1.0});
          }
          if (slot_b) {
            gd.b_first = (int)ops.size();
            gd.b_count = 1;
            ops.push_back({pl.dxb + slot * pl.nq_pad, pl.dkb, 0, 1.0});
          }
        } else {
          gd.a_first = ua.a_first;
          gd.a_count = ua.a_count;
          gd.b_first = ub.a_first;
          gd.b_count = ub.a_count;
        }
        gterms[slot] = gd;
        uA[slot] = ua;
        uB[slot] = ub;
      }
      // accumulate lists: per quadrant, (slot, sign) in term order
      std::vector<int32_t> lstart(pl.nquads + 1, 0), lslot;
      std::vector<double> lsign;
      std::vector<int64_t> rstart(pl.nquads), cstart(pl.nquads);
      for (int q = 0; q < pl.nquads; ++q) {
        lstart[q] = (int32_t)lslot.size();
        for (int t = t0; t < t1; ++t)
          for (const Op &op : pl.terms[pl.seq[t]].c)
            if (op.q == q) {
              lslot.push_back(t - t0);
              lsign.push_back((double)op.s);
            }
        int64_t r, c;
        quad_rc(q, pl.level, r, c);
        rstart[q] = pl.cr + r * pl.mq_pad;
        cstart[q] = pl.cc + c * pl.nq_pad;
      }
      lstart[pl.nquads] = (int32_t)lslot.size();
      char *tab = cw + pl.off_tab + (size_t)bi * pl.tab_bytes;
      std::vector<char> host(pl.tab_bytes, 0);
      size_t o = 0;
      auto put = [&](const void *src, size_t bytes) {
        memcpy(host.data() + o, src, bytes);
        const size_t at = o;
        o += bytes;
        return tab + at;
      };
      Batch b{};
      b.t0 = t0;
      b.t1 = t1;
      b.d_g = reinterpret_cast<const TermDesc *>(put(gterms.data(), nb * sizeof(TermDesc)));
      b.d_ua = reinterpret_cast<const TermDesc *>(put(uA.data(), nb * sizeof(TermDesc)));
      b.d_ub = reinterpret_cast<const TermDesc *>(put(uB.data(), nb * sizeof(TermDesc)));
      b.d_ops = reinterpret_cast<const OpDesc *>(put(ops.data(), ops.size() * sizeof(OpDesc)));
      if (o > pl.tab_bytes) return fail(STC_EINVAL, "internal: table overflow");
      if (!restored)
        if (int rc = upload(host.data(), o, tab, s)) return rc;
      char *acc = cw + pl.off_acc + (size_t)bi * pl.acc_bytes;
      std::vector<char> hacc(pl.acc_bytes, 0);
      size_t ao = 0;
      auto aput = [&](const void *src, size_t bytes, size_t slot_bytes) {
        memcpy(hacc.data() + ao, src, bytes);
        const size_t at = ao;
        ao += align256(slot_bytes);
        return acc + at;
      };
      AccArgs &aa = b.aa;
      aa.c_ready = c_ready;
      aa.list_start = reinterpret_cast<const int32_t *>(aput(lstart.data(), lstart.size() * 4, (pl.nquads + 1) * 4));
      aa.list_slot = reinterpret_cast<const int32_t *>(
          aput(lslot.data(), lslot.size() * 4, (size_t)pl.batch * pl.nquads * 4));
      aa.list_sign = reinterpret_cast<const double *>(
          aput(lsign.data(), lsign.size() * 8, (size_t)pl.batch * pl.nquads * 8));
      aa.row_start = reinterpret_cast<const int64_t *>(aput(rstart.data(), rstart.size() * 8, pl.nquads * 8));
      aa.col_start = reinterpret_cast<const int64_t *>(aput(cstart.data(), cstart.size() * 8, pl.nquads * 8));
      if (!restored)
        if (int rc = upload(hacc.data(), pl.acc_bytes, acc, s)) return rc;
      aa.M = M;
      aa.m_ld = pl.nq_pad;
      aa.m_stride = pl.m_slot;
      aa.C = C;
      aa.pool = pool;
      aa.mq = pl.mq;
      aa.nq = pl.nq;
      aa.nquads = pl.nquads;
      aa.max_list = 0;
      for (int q = 0; q < pl.nquads; ++q) aa.max_list = std::max(aa.max_list, lstart[q + 1] - lstart[q]);
      b.nupd = (int64_t)lslot.size();
      batches.push_back(b);
    }
    // the fused set-up shared by the batches: maps, coordinates, repacked operands
    GemmArgs gf_ab = g;
    CUtensorMap maps_ab[3];
    int fused_ab = 0;
    if (slots) {  // per-term slots (regular by construction) and, one-sided, the other side's views
      CoordJobs jobs{};
      if (plan_fused(p, pl, mixed_sides(p, pl), slot_a ? PA : A, slot_b ? PB : B, nullptr, gf_ab, maps_ab, jobs)) {
        gf_ab.A = slot_a ? PA : A;
        gf_ab.B = slot_b ? PB : B;
        gf_ab.coords = coords;
        if (!restored) {
          CU(launch_pool_coords(pool, coords, jobs, s), "k_pool_coords");
          ++launches;
        }
        fused_ab = 1;
      }
    } else {
      fused_ab = prepare_fused(gf_ab, maps_ab, nullptr);
      if (fused_ab < 0) return -fused_ab;
    }
    if (int rc = save_snapshot()) return rc;
    // pass 2: per batch the operand slots, the DMMA launch, the accumulate
    for (int bi = 0; bi < pl.nbatches; ++bi) {
      const Batch &b = batches[bi];
      const int nb = b.t1 - b.t0;
      if (slots && pl.presum) {
        // one pass per side: every element position's 4^L quadrant values -> the batch's sums
        if (presum_runs) {
          PresumArgs pa = presum_args(pl, 0, A, slot_a && !skip_a ? PA : nullptr, pool, b.t0, b.t1);
          if (bi == 0 && zero) {
            pa.zero = zero;
            pa.zero_words = zero_words;
          }
          CU(launch_presum2(pa, presum_args(pl, 1, B, slot_b && !skip_b ? PB : nullptr, pool, b.t0, b.t1), s),
             "k_presum");
          ++launches;
        }
        if (shared_slots && ovr->after_presum) CU(cudaEventRecord(ovr->after_presum, s), "cudaEventRecord");
      } else if (slots) {
        UnpackArgs ua{};
        ua.pool = pool;
        ua.ops = b.d_ops;
        ua.nterms = nb;
        ua.D = A;
        ua.out = PA;
        ua.terms = b.d_ua;
        ua.x_len = pl.mq_pad;
        ua.k_len = pl.kq_pad;
        ua.slot_stride = pl.pa_slot;
        ua.kfast = pl.a_kfast;
        CU(launch_unpack(ua, s), "k_unpack(A)");
        ua.D = B;
        ua.out = PB;
        ua.terms = b.d_ub;
        ua.x_len = pl.nq_pad;
        ua.slot_stride = pl.pb_slot;
        ua.kfast = pl.b_kfast;
        CU(launch_unpack(ua, s), "k_unpack(B)");
        launches += 2;
        st.slow_blocks += 2 * nb;
      }
      GemmArgs gb = g;
      gb.A = slot_a ? PA : A;
      gb.B = slot_b ? PB : B;
      gb.C = nullptr;
      gb.terms = b.d_g;
      gb.ops = b.d_ops;
      gb.tgts = nullptr;
      gb.nterms = nb;
      gb.total_items = (int)(P * nb);
      gb.a_kfast = pl.a_kfast;  // Naive slots follow the source orientation too
      gb.b_kfast = pl.b_kfast;
      gb.dense_out = 1;
      gb.use_tickets = 0;
      gb.M = M;
      gb.m_ld = pl.nq_pad;
      gb.m_stride = pl.m_slot;
      gb.counter = counters + bi;
      const int grid = (int)std::min<int64_t>(pl.grid, gb.total_items);
      GemmArgs gf = gb;
      if (fused_ab) {  // per-batch fields over the fused set-up (maps, coordinates, packed operands)
        const GemmArgs &base = gf_ab;
        gf.A = base.A;
        gf.B = base.B;
        gf.a_kfast = base.a_kfast;
        gf.b_kfast = base.b_kfast;
        gf.coords = base.coords;
        gf.umax = base.umax;
        gf.one_view = base.one_view;
        gf.stages = base.stages;
        gf.stage_dbl = base.stage_dbl;
        gf.tshape = base.tshape;
        gf.psum = base.psum;
        gf.kchunks = base.kchunks;
        gf.cred = 0;
        for (int sd = 0; sd < 3; ++sd) {
          gf.tm_rank[sd] = base.tm_rank[sd];
          for (int d = 0; d < 5; ++d) gf.tm_src[sd][d] = base.tm_src[sd][d];
          for (int part = 0; part < 2; ++part) {
            gf.tm_np[sd][part] = base.tm_np[sd][part];
            for (int i = 0; i < 4; ++i) gf.tm_pstr[sd][part][i] = base.tm_pstr[sd][part][i];
          }
        }
      }
      if (ev_before && bi == 0) CU(cudaEventRecord(ev_before, s), "cudaEventRecord");
      if (fused_ab) {
        tma = !packed;  // TMA boxes of the operands or of their packed slots (the reference's Naive GEMM: dense, fast blocks)
        CU(launch_fused(gf, grid, s, maps_ab), "k_strassen_fused(dense)");
      } else {
        if (pl.tshape != 0) return fail(STC_EINVAL, "internal: tile shape %d needs the fused kernel", pl.tshape);
        CU(launch_gemm(gb, grid, s), "k_strassen_gemm(dense)");
      }
      if (ev_after && bi == pl.nbatches - 1) CU(cudaEventRecord(ev_after, s), "cudaEventRecord");
      CU(launch_accumulate(b.aa, s), "k_accumulate");
      launches += 2;
      st.slow_updates += b.nupd;
    }
  }
  st.total_flops = 2.0 * (double)pl.tm * (double)pl.tn * (double)pl.kq_pad * (double)P * (double)T;
  // operand blocks (one view of one side x one k-chunk per tile): TMA-staged
  // boxes are the reference's fast (constant-stride) blocks
  (tma ? st.fast_blocks : st.slow_blocks) += 2 * (int64_t)(pl.kq_pad / BK) * P * T;
  st.leaf_multiplies = T;
  st.work_items = P * T;
  st.kernel_launches = launches + g_stage_launches;
  st.pieces = 1;
  if (stats) *stats = st;
  return STC_OK;
}

// Problems up to this many executed flops replay a CUDA graph of their launch
// sequence (~0.1 ms of DMMA work: the host's per-call work is then comparable).
constexpr double kGraphFlops = 4e9;

// Per thread and device: the non-blocking stream graphs are captured on.
static cudaStream_t capture_stream(int dev) {
  thread_local std::vector<cudaStream_t> streams;
  if (dev < 0) return nullptr;
  if ((int)streams.size() <= dev) streams.resize(dev + 1, nullptr);
  if (!streams[dev] && cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    streams[dev] = nullptr;
  }
  return streams[dev];
}

int stc_contract(const stc_problem *p, const double *A, const double *B, double *C, void *workspace,
                 size_t workspace_bytes, void *stream, stc_stats *stats) {
  env_refresh();
  std::shared_ptr<const Plan> plan;
  const int grid_hint = gemm_max_grid(MAX_OPS);
  if (grid_hint <= 0) return fail(STC_ECUDA, "could not size the DMMA grid");
  if (int rc = cached_plan(p, plan, grid_hint)) return rc;
  const Plan &pl = *plan;
  if (!A || !B || !C) return fail(STC_EINVAL, "null operand pointer");
  if (!workspace || workspace_bytes < pl.total)
    return fail(STC_EWORKSPACE, "workspace too small: need %zu bytes, got %zu", pl.total, workspace_bytes);
  if (reinterpret_cast<uintptr_t>(workspace) & 255) return fail(STC_EINVAL, "workspace must be 256-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char *ws = reinterpret_cast<char *>(workspace);
  const int32_t *c_ready = g_c_ready;  // consumed by this call, like the kernel events
  g_c_ready = nullptr;
  cudaEvent_t ev_before = g_ev_before, ev_after = g_ev_after;
  g_ev_before = g_ev_after = nullptr;
  SlotOverride ovr_v = g_slot_ovr;
  const SlotOverride *ovr = g_slot_ovr_set ? &ovr_v : nullptr;
  g_slot_ovr_set = false;
  g_slot_ovr = SlotOverride{};
  int dev = 0;
  CU(cudaGetDevice(&dev), "cudaGetDevice");
  Resident *res = pl.res.get();

  // Small problems: replay the graph captured for these pointers (the operand mode
  // below is a function of the plan and the pointers, so the key implies it).
  const double flops = 2.0 * (double)pl.tm * (double)pl.tn * (double)pl.kq_pad *
                       (double)((pl.mq_pad / pl.tm) * (pl.nq_pad / pl.tn)) * (double)pl.terms.size();
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  const bool graphs = res && !ev_before && !ev_after && !c_ready && !ovr && flops <= kGraphFlops && !stc_env("STC_NO_GRAPH") &&
                      !stc_env("STC_NO_SNAPSHOT") && cudaStreamIsCapturing(s, &cap) == cudaSuccess &&
                      cap == cudaStreamCaptureStatusNone;
  const GraphKey key{A, B, C, ws, dev, 0};
  if (graphs) {
    stc_stats gst{};
    if (res->replay(key, s, gst)) {
      if (stats) *stats = gst;
      return STC_OK;
    }
  }

  // Operand mode: per-term slots (Naive, pre-summed), the operands' own TMA views, or
  // their repacked quadrant blocks (one gather pass per operand, pure copies).
  const bool slots = pl.variant == STC_VARIANT_NAIVE || pl.presum;
  bool direct = false;
  if (!slots) {
    GemmArgs gt{};
    CUtensorMap mt[3];
    CoordJobs jt{};
    direct = plan_fused(p, pl, direct_sides(p, pl), A, B, pl.ticketed ? C : nullptr, gt, mt, jt);
  }
  const bool packed = !slots && !direct && pl.need_pack;

  // The constant region of the workspace -- scatter vectors, chunk strides, map
  // coordinates, term / op / target tables, accumulate lists, zeroed tickets and
  // counters -- depends only on the plan (and the operand mode): the first call of a
  // plan builds it and keeps a device snapshot; later calls restore it with one
  // kernel instead of 5-10 small launches (Resident).
  const int mode = packed ? 1 : 0;
  const void *snap = res ? res->ready(mode, dev, s) : nullptr;
  // the graph is captured on a private stream (the caller's may be the legacy default
  // stream, which cannot capture) and launched on the caller's
  cudaStream_t cs = capture_stream(dev);
  if (graphs && snap && cs && cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
    stc_stats st{};
    const int rc =
        contract_run(p, pl, A, B, C, ws, cs, nullptr, nullptr, nullptr, direct, packed, mode, dev, snap, nullptr, &st);
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(cs, &graph);
    cudaGraphExec_t exec = nullptr;
    const bool ok = rc == STC_OK && ec == cudaSuccess && graph &&
                    cudaGraphInstantiateWithFlags(&exec, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    if (ok) {
      if (cudaGraphLaunch(exec, s) != cudaSuccess) {
        cudaGraphExecDestroy(exec);
        return cuda_fail(cudaGetLastError(), "cudaGraphLaunch");
      }
      GraphKey k = key;
      k.mode = mode;
      res->keep(k, exec, st);
      if (stats) *stats = st;
      return STC_OK;
    }
    cudaGetLastError();  // nothing ran: fall through to direct launches
    if (rc != STC_OK && ec == cudaSuccess) return rc;
  }
  return contract_run(p, pl, A, B, C, ws, s, c_ready, ev_before, ev_after, direct, packed, mode, dev, snap, ovr,
                      stats);
}

int stc_bundle_scatter(const stc_bundle *bundle, int64_t base, int64_t out_len, int64_t *out, void *stream) {
  if (!bundle || !out) return fail(STC_EINVAL, "null argument");
  if (int rc = check_bundle(*bundle, "bundle")) return rc;
  const int64_t len = bundle_len(*bundle);
  if (out_len < len) return fail(STC_EINVAL, "out_len %lld shorter than the bundle (%lld)", (long long)out_len, (long long)len);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Tiling none;
  VecDesc d = vec_bundle(*bundle, base, 1, 1, none);
  d.q_len = out_len;  // entries beyond len read PAD
  d.q_len_pad = out_len;
  d.out_start = 0;
  VecDesc *dd = nullptr;
  CU(cudaMallocAsync(reinterpret_cast<void **>(&dd), sizeof(VecDesc), s), "cudaMallocAsync");
  if (int rc = upload(&d, sizeof(d), dd, s)) return rc;
  CU(launch_build_pool(dd, 1, out_len, out, s), "k_build_pool");
  CU(cudaFreeAsync(dd, s), "cudaFreeAsync");
  return STC_OK;
}

int stc_block_vector(const int64_t *scat, int64_t len, int64_t blk, int64_t unit_stride, int64_t *out,
                     void *stream) {
  if (blk < 1) return fail(STC_EINVAL, "block sizes must be >= 1");
  if (len < 0 || (len > 0 && (!scat || !out))) return fail(STC_EINVAL, "bad scatter vector");
  CU(launch_block_vector(scat, len, blk, unit_stride, out, reinterpret_cast<cudaStream_t>(stream)), "k_block_vector");
  return STC_OK;
}

int stc_fused_term_workspace_size(int64_t m, int64_t n, int64_t k, int n_a, int n_b, int n_c, size_t *bytes) {
  env_refresh();
  if (m < 1 || n < 1 || k < 1) return fail(STC_EINVAL, "empty fused term %lldx%lldx%lld", (long long)m, (long long)n, (long long)k);
  if (n_a < 1 || n_b < 1 || n_c < 1 || n_a > MAX_OPS || n_b > MAX_OPS || n_c > MAX_OPS)
    return fail(STC_EINVAL, "need 1..%d views per side", MAX_OPS);
  const int64_t mp = rup(m, BM), np = rup(n, BN), kp = rup(k, BK);
  size_t pool = (size_t)(n_a * (mp + kp) + n_b * (np + kp) + n_c * (mp + np)) * 8;
  size_t tab = sizeof(TermDesc) + (size_t)(n_a + n_b) * sizeof(OpDesc) + (size_t)n_c * sizeof(TgtDesc);
  if (bytes) *bytes = align256(pool) + align256(pool / BK) + align256(tab) + 256;  // pool, kbs, tables, counter
  return STC_OK;
}

int stc_fused_term(int64_t m, int64_t n, int64_t k, const double *A, int n_a, const int64_t *const *a_rows,
                   const int64_t *const *a_cols, const double *a_coeffs, const double *B, int n_b,
                   const int64_t *const *b_rows, const int64_t *const *b_cols, const double *b_coeffs, double *C,
                   int n_c, const int64_t *const *c_rows, const int64_t *const *c_cols, const double *c_coeffs,
                   uint32_t flags, void *workspace, size_t workspace_bytes, void *stream, stc_stats *stats) {
  env_refresh();
  size_t need = 0;
  if (int rc = stc_fused_term_workspace_size(m, n, k, n_a, n_b, n_c, &need)) return rc;
  if (!workspace || workspace_bytes < need)
    return fail(STC_EWORKSPACE, "workspace too small: need %zu bytes, got %zu", need, workspace_bytes);
  for (int i = 0; i < n_a; ++i)
    if (a_coeffs[i] != 1.0 && a_coeffs[i] != -1.0) return fail(STC_EINVAL, "coefficients must be +/-1");
  for (int i = 0; i < n_b; ++i)
    if (b_coeffs[i] != 1.0 && b_coeffs[i] != -1.0) return fail(STC_EINVAL, "coefficients must be +/-1");
  for (int i = 0; i < n_c; ++i)
    if (c_coeffs[i] != 1.0 && c_coeffs[i] != -1.0) return fail(STC_EINVAL, "coefficients must be +/-1");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char *ws = reinterpret_cast<char *>(workspace);
  int64_t *pool = reinterpret_cast<int64_t *>(ws);
  const int64_t mp = rup(m, BM), np = rup(n, BN), kp = rup(k, BK);
  int64_t at = 0;
  std::vector<OpDesc> ops;
  std::vector<TgtDesc> tg;
  auto put = [&](const int64_t *src, int64_t len, int64_t lenp) {
    const int64_t start = at;
    at += lenp;
    return std::make_pair(start, launch_copy_pad(src, len, lenp, pool + start, s));
  };
  for (int i = 0; i < n_a; ++i) {
    auto x = put(a_rows[i], m, mp), kk = put(a_cols[i], k, kp);
    CU(x.second, "copy_pad");
    CU(kk.second, "copy_pad");
    ops.push_back({x.first, kk.first, 0, a_coeffs[i]});
  }
  for (int i = 0; i < n_b; ++i) {
    auto x = put(b_cols[i], n, np), kk = put(b_rows[i], k, kp);
    CU(x.second, "copy_pad");
    CU(kk.second, "copy_pad");
    ops.push_back({x.first, kk.first, 0, b_coeffs[i]});
  }
  for (int i = 0; i < n_c; ++i) {
    auto r = put(c_rows[i], m, mp), c = put(c_cols[i], n, np);
    CU(r.second, "copy_pad");
    CU(c.second, "copy_pad");
    TgtDesc t{};
    t.row_start = r.first;
    t.col_start = c.first;
    t.sign = c_coeffs[i];
    tg.push_back(t);
  }
  TermDesc td{};
  td.a_first = 0;
  td.a_count = n_a;
  td.b_first = n_a;
  td.b_count = n_b;
  td.c_first = 0;
  td.c_count = n_c;
  int64_t *kbs = reinterpret_cast<int64_t *>(ws + align256((size_t)at * 8));
  CU(launch_chunk_strides(pool, at / BK, kbs, s), "k_chunk_strides");
  char *tab = ws + align256((size_t)at * 8) + align256((size_t)(at / BK) * 8);
  std::vector<char> host(sizeof(TermDesc) + ops.size() * sizeof(OpDesc) + tg.size() * sizeof(TgtDesc) + 8);
  size_t o = 0;
  memcpy(host.data() + o, &td, sizeof(td));
  o += sizeof(td);
  memcpy(host.data() + o, ops.data(), ops.size() * sizeof(OpDesc));
  o += ops.size() * sizeof(OpDesc);
  memcpy(host.data() + o, tg.data(), tg.size() * sizeof(TgtDesc));
  o += tg.size() * sizeof(TgtDesc);
  // counter lives after the tables
  char *ctr = tab + align256(o);
  if (ctr + 4 > ws + workspace_bytes) return fail(STC_EWORKSPACE, "workspace too small for counters");
  g_stage_launches = 0;
  if (int rc = upload(host.data(), o, tab, s, ctr, 4)) return rc;
  GemmArgs g{};
  g.A = A;
  g.B = B;
  g.C = C;
  g.pool = pool;
  g.terms = reinterpret_cast<const TermDesc *>(tab);
  g.ops = reinterpret_cast<const OpDesc *>(tab + sizeof(TermDesc));
  g.tgts = reinterpret_cast<const TgtDesc *>(tab + sizeof(TermDesc) + ops.size() * sizeof(OpDesc));
  g.nterms = 1;
  g.tiles_m = (int)(mp / BM);
  g.tiles_n = (int)(np / BN);
  g.kchunks = (int)(kp / BK);
  g.total_items = g.tiles_m * g.tiles_n;
  g.a_kfast = 0;
  g.b_kfast = 0;
  g.dense_out = 0;
  g.use_tickets = 0;
  g.group_m = 8;
  g.max_ops = std::max(n_a, n_b);
  g.nraw = gemm_nraw(g.max_ops);
  g.kwin = gemm_kwin(g.max_ops);
  g.kbs = kbs;
  g.force_slow = (flags & STC_FLAG_FORCE_SLOW) ? 1 : 0;
  g.counter = reinterpret_cast<int32_t *>(ctr);
  const int grid = std::min(gemm_max_grid(MAX_OPS), g.total_items);
  CU(launch_gemm(g, grid, s), "k_strassen_gemm(fused_term)");
  if (stats) {
    stc_stats st{};
    st.total_flops = 2.0 * BM * BN * (double)kp * (double)g.total_items;
    st.slow_blocks = 2 * (int64_t)g.kchunks * g.total_items;
    st.slow_updates = (int64_t)g.total_items * n_c;
    st.leaf_multiplies = 1;
    st.work_items = g.total_items;
    st.kernel_launches = 2 * (n_a + n_b + n_c) + 2 + g_stage_launches;  // copy_pad per vector, chunk strides, gemm
    *stats = st;
  }
  (void)flags;
  return STC_OK;
}

int stc_accumulate_dense(const double *M, int64_t ldm, int64_t m, int64_t n, double *C, const int64_t *rows,
                         const int64_t *cols, double coeff, void *stream, stc_stats *stats) {
  if (m < 0 || n < 0 || ldm < m) return fail(STC_EINVAL, "matrix shape (%lld, %lld) / ld %lld invalid", (long long)m, (long long)n, (long long)ldm);
  CU(launch_accum_dense_single(M, ldm, m, n, C, rows, cols, coeff, reinterpret_cast<cudaStream_t>(stream)),
     "k_accum_dense_single");
  if (stats) {
    stc_stats st{};
    st.slow_updates = 1;
    st.kernel_launches = 1;
    *stats = st;
  }
  return STC_OK;
}

int stc_unpack_sum(double *out, int64_t ldo, int64_t m, int64_t n, const double *data, int nviews,
                   const int64_t *const *rows, const int64_t *const *cols, const double *coeffs, void *stream,
                   stc_stats *stats) {
  if (nviews < 1 || nviews > MAX_OPS) return fail(STC_EINVAL, "need 1..%d views", MAX_OPS);
  if (m < 0 || n < 0 || ldo < m) return fail(STC_EINVAL, "out must be a float64 %lldx%lld matrix", (long long)m, (long long)n);
  ViewSet vs{};
  vs.n = nviews;
  for (int i = 0; i < nviews; ++i) {
    vs.rows[i] = rows[i];
    vs.cols[i] = cols[i];
    vs.coeff[i] = coeffs[i];
  }
  CU(launch_unpack_views(out, ldo, m, n, data, vs, reinterpret_cast<cudaStream_t>(stream)), "k_unpack_views");
  if (stats) {
    stc_stats st{};
    st.slow_blocks = 1;
    st.kernel_launches = 1;
    *stats = st;
  }
  return STC_OK;
}

namespace {
// fast / slow counts of the component passes: written by the kernel into page-locked
// host memory (one 16-byte block per thread, kept), read after a stream synchronise
int64_t *host_counts() {
  thread_local int64_t *p = nullptr;
  if (!p && cudaHostAlloc(reinterpret_cast<void **>(&p), 2 * sizeof(int64_t), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    p = nullptr;
  }
  return p;
}
}  // namespace

int stc_pack_panel(int side, const double *data, int nviews, const int64_t *const *rows, const int64_t *const *cols,
                   const int64_t *const *rbs, const int64_t *const *cbs, const double *coeffs, int64_t x0,
                   int64_t xcount, int64_t k0, int64_t kcount, int64_t width, int64_t kblock, uint32_t flags,
                   double *out, int64_t out_depth, void *stream, stc_stats *stats) {
  if (side != 0 && side != 1) return fail(STC_EINVAL, "side must be 0 (A) or 1 (B)");
  if (nviews < 1 || nviews > MAX_OPS) return fail(STC_EINVAL, "need 1..%d views", MAX_OPS);
  if (!data || !rows || !cols || !coeffs || !out) return fail(STC_EINVAL, "null argument");
  if (x0 < 0 || xcount < 0 || k0 < 0 || kcount < 0 || width < 1 || kblock < 1 || out_depth < kcount)
    return fail(STC_EINVAL, "block [%lld,+%lld) x [%lld,+%lld), width %lld, k block %lld, depth %lld invalid",
                (long long)x0, (long long)xcount, (long long)k0, (long long)kcount, (long long)width,
                (long long)kblock, (long long)out_depth);
  if (x0 % width || k0 % kblock) return fail(STC_EINVAL, "block origin must be a multiple of the register block");
  const bool count = stats && rbs && cbs;
  PanelArgs a{};
  a.vs.n = nviews;
  for (int t = 0; t < nviews; ++t) {
    if (coeffs[t] != 1.0 && coeffs[t] != -1.0) return fail(STC_EINVAL, "coefficients must be +/-1");
    a.vs.rows[t] = rows[t];
    a.vs.cols[t] = cols[t];
    a.vs.coeff[t] = coeffs[t];
    if (count) {
      a.xbs[t] = side == 0 ? rbs[t] : cbs[t];
      a.kbs[t] = side == 0 ? cbs[t] : rbs[t];
    }
  }
  a.side = side;
  a.x0 = x0, a.xcount = xcount, a.k0 = k0, a.kcount = kcount, a.width = width, a.kblock = kblock, a.depth = out_depth;
  a.force_slow = (flags & STC_FLAG_FORCE_SLOW) ? 1 : 0;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int64_t *cnt = count ? host_counts() : nullptr;
  if (count && !cnt) return fail(STC_ECUDA, "cudaHostAlloc(counters) failed");
  CU(launch_pack_panel(a, data, out, cnt, s), "k_pack_panel");
  if (stats) {
    stc_stats st{};
    st.kernel_launches = count ? 2 : 1;
    if (count) {
      CU(cudaStreamSynchronize(s), "cudaStreamSynchronize");
      st.fast_blocks = cnt[0];
      st.slow_blocks = cnt[1];
    }
    *stats = st;
  }
  return STC_OK;
}

int stc_microtile(const double *a_sliver, int64_t lda, const double *b_sliver, int64_t ldb, int64_t k, int mr, int nr,
                  double *C, int n_targets, const int64_t *const *rows, const int64_t *const *cols,
                  const int64_t *const *rbs, const int64_t *const *cbs, const double *coeffs, const int64_t *i0,
                  const int64_t *j0, const int64_t *m, const int64_t *n, uint32_t flags, void *stream,
                  stc_stats *stats) {
  if (stats) *stats = stc_stats{};
  if (k == 0) return STC_OK;  // the reference returns before touching the targets (kernels.py:211-212)
  if (k < 0 || mr < 1 || nr < 1 || (int64_t)mr * nr > 4096 || lda < k || ldb < nr)
    return fail(STC_EINVAL, "tile %d x %d, depth %lld, lda %lld, ldb %lld invalid", mr, nr, (long long)k,
                (long long)lda, (long long)ldb);
  if (n_targets < 0 || n_targets > MAX_OPS) return fail(STC_EINVAL, "at most %d targets", MAX_OPS);
  if (!a_sliver || !b_sliver || (n_targets && (!C || !rows || !cols || !coeffs || !i0 || !j0 || !m || !n)))
    return fail(STC_EINVAL, "null argument");
  const bool count = stats && rbs && cbs;
  TileTargets t{};
  t.n_targets = n_targets;
  for (int g = 0; g < n_targets; ++g) {
    if (i0[g] % mr || j0[g] % nr) return fail(STC_EINVAL, "tile origin must be block-aligned");
    if (i0[g] < 0 || j0[g] < 0 || i0[g] >= m[g] || j0[g] >= n[g])
      return fail(STC_EINVAL, "tile origin (%lld, %lld) outside the %lld x %lld target", (long long)i0[g],
                  (long long)j0[g], (long long)m[g], (long long)n[g]);
    t.rows[g] = rows[g], t.cols[g] = cols[g];
    t.rbs[g] = count ? rbs[g] : nullptr, t.cbs[g] = count ? cbs[g] : nullptr;
    t.coeff[g] = coeffs[g];
    t.i0[g] = i0[g], t.j0[g] = j0[g], t.m[g] = m[g], t.n[g] = n[g];
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int64_t *cnt = count ? host_counts() : nullptr;
  if (count && !cnt) return fail(STC_ECUDA, "cudaHostAlloc(counters) failed");
  CU(launch_microtile(a_sliver, lda, b_sliver, ldb, k, mr, nr, C, t, (flags & STC_FLAG_FORCE_SLOW) ? 1 : 0, cnt, s),
     "k_microtile");
  if (stats) {
    stats->kernel_launches = 1;
    stats->total_flops = 2.0 * mr * nr * (double)k;
    if (count) {
      CU(cudaStreamSynchronize(s), "cudaStreamSynchronize");
      stats->fast_updates = cnt[0];
      stats->slow_updates = cnt[1];
    }
  }
  return STC_OK;
}

int stc_sq_norms(int ndim, const int64_t *extents, const double *x, const int64_t *x_strides, int64_t x_base,
                 const double *ref, const int64_t *ref_strides, int64_t ref_base, double *out, void *stream) {
  if (ndim < 0 || ndim > STC_MAX_LABELS) return fail(STC_EINVAL, "bad rank %d", ndim);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nblocks = 148 * 4;
  double *part = nullptr;
  CU(cudaMallocAsync(reinterpret_cast<void **>(&part), sizeof(double) * 2 * nblocks, s), "cudaMallocAsync");
  CU(launch_sq_norms(ndim, extents, x, x_strides, x_base, ref, ref_strides, ref_base, part, nblocks, s), "k_sq_norms");
  std::vector<double> h(2 * nblocks);
  CU(cudaMemcpyAsync(h.data(), part, sizeof(double) * 2 * nblocks, cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync");
  CU(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  CU(cudaFreeAsync(part, s), "cudaFreeAsync");
  double a = 0.0, b = 0.0;
  for (int i = 0; i < nblocks; ++i) {
    a += h[2 * i];
    b += h[2 * i + 1];
  }
  out[0] = a;
  out[1] = b;
  return STC_OK;
}

int stc_fill_uniform(double *out, int ndim, const int64_t *extents, const int64_t *strides, int64_t base,
                     uint64_t seed, void *stream) {
  if (ndim < 0 || ndim > STC_MAX_LABELS) return fail(STC_EINVAL, "bad rank %d", ndim);
  if (!out) return fail(STC_EINVAL, "null output");
  for (int d = 0; d < ndim; ++d)
    if (extents[d] < 0) return fail(STC_EINVAL, "negative extents");
  CU(launch_fill_uniform(out, ndim, extents, strides, base, seed, reinterpret_cast<cudaStream_t>(stream)),
     "k_fill_uniform");
  return STC_OK;
}

int stc_plan_describe(const stc_problem *p, int grid, stc_plan_info *info) {
  if (!info) return fail(STC_EINVAL, "null info");
  std::shared_ptr<const Plan> plan;
  if (grid <= 0) grid = 148;
  if (int rc = cached_plan(p, plan, grid)) return rc;
  const Plan &pl = *plan;
  memset(info, 0, sizeof(*info));
  info->ticketed = pl.ticketed;
  info->presum = pl.presum;
  info->presum_sides = pl.presum ? pl.presum_sides : 0;
  info->need_pack = pl.need_pack;
  info->tshape = pl.tshape;
  info->batch = pl.batch;
  info->nbatches = pl.nbatches;
  info->terms = (int32_t)pl.terms.size();
  info->tiles = (int64_t)(pl.mq_pad / pl.tm) * (pl.nq_pad / pl.tn);
  info->mq_pad = pl.mq_pad;
  info->nq_pad = pl.nq_pad;
  info->kq_pad = pl.kq_pad;
  info->workspace = pl.total;
  if (pl.variant != STC_VARIANT_NAIVE && !pl.presum) {
    GemmArgs g{};
    CUtensorMap maps[3];
    CoordJobs jobs{};
    info->fused_direct = plan_fused(p, pl, direct_sides(p, pl), nullptr, nullptr, nullptr, g, maps, jobs);
  }
  info->c_boxes = c_boxes_regular(p, pl.ti, pl.tj, pl.level);
  return STC_OK;
}

int stc_shard_problem(const stc_problem *p, int world, int rank, int label, stc_problem *out, int64_t *start,
                      int64_t *stop, int32_t *label_out) {
  if (!p || !out) return fail(STC_EINVAL, "null argument");
  if (world < 1) return fail(STC_EINVAL, "world size must be positive");
  if (rank < 0 || rank >= world) return fail(STC_EINVAL, "rank %d outside [0, %d)", rank, world);
  const stc_bundle &cj = p->c_col;
  if (cj.nlab == 0) return fail(STC_EINVAL, "the J bundle is empty: nothing to split");
  if (label < 0) {  // shard.plan_shards' default: divisible extents first, then the largest C stride
    int best = -1;
    for (int d = 0; d < cj.nlab; ++d) {
      if (cj.ext[d] < world) continue;
      const bool div = cj.ext[d] % world == 0;
      if (best < 0) {
        best = d;
        continue;
      }
      const bool bdiv = cj.ext[best] % world == 0;
      const int64_t s = cj.str[d] < 0 ? -cj.str[d] : cj.str[d], bs = cj.str[best] < 0 ? -cj.str[best] : cj.str[best];
      if (div > bdiv || (div == bdiv && s > bs)) best = d;
    }
    if (best < 0) return fail(STC_EINVAL, "no J label has extent >= %d", world);
    label = best;
  }
  if (label >= cj.nlab) return fail(STC_EINVAL, "label %d is not in the J bundle", label);
  const int64_t ext = cj.ext[label], base = ext / world, extra = ext % world;
  const int64_t s0 = rank * base + std::min<int64_t>(rank, extra);
  const int64_t n = base + (rank < extra ? 1 : 0);
  if (n < 1) return fail(STC_EINVAL, "rank %d gets an empty range of label %d", rank, label);
  *out = *p;
  out->b_col.ext[label] = n;
  out->c_col.ext[label] = n;
  out->b_base += s0 * p->b_col.str[label];
  out->c_base += s0 * p->c_col.str[label];
  if (start) *start = s0;
  if (stop) *stop = s0 + n;
  if (label_out) *label_out = label;
  return STC_OK;
}

}  // extern "C"
