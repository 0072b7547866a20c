// stc_host.cu -- host-operand entry point (stc_contract_host): the
// contraction of tensors that live in host memory, with the PCIe transfers
// pipelined against the DMMA work.
//
// The reference computes on host arrays in place (strassen.contract,
// strassen.py:141-207).  On the B200 the operands must cross PCIe, which
// costs about twice the FP64 tensor-core time of the contraction itself
// (cfg2: 0.4 GB in, 0.13 GB out).  Instead of upload -> compute -> download,
// the problem is cut along one label of the I or J bundle into S pieces:
//
//   C[:, J_s] += A . B[:, J_s]     (J split; the I split is symmetric)
//
// Each piece is an independent contraction over the same block-scatter
// views, run by stc_contract with the piece's extent and base offset (the
// piece is itself an L-level Strassen contraction; the multi-GPU shard path
// splits the same way, shard.py).  Streams:
//   h2d:      shared operand, then (operand piece, C piece) for s = 0..S-1
//   comp[2]:  piece s on comp[s % 2] after its inputs arrived; alternating
//             streams let piece s+1's CTAs fill the SMs of piece s's tail
//   d2h:      C piece s as soon as piece s finished
// so the copy engines and the tensor cores run concurrently and the call
// costs about max(H2D) + one piece's compute + one piece's download.
//
// Copies are 2-D (cudaMemcpy2DAsync): in a compact tensor (strides a
// permutation of a dense layout) restricting one label to a range is a set of
// equal-length runs at a fixed pitch.  The split label is chosen so the runs
// are long in both tensors it touches; when no label qualifies (small
// problem, non-compact storage, short runs) S = 1 and the call is the plain
// upload -> contract -> download sequence on the same streams.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "stc_internal.cuh"

using namespace stc;

namespace {

int herr(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
int herr(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return set_error(code, buf);
}

#define HCU(expr, what)                                                                     \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess) return herr(STC_ECUDA, "CUDA error in %s: %s", what, cudaGetErrorString(_e)); \
  } while (0)

constexpr int64_t kMinRunBytes = 4096;          // shortest copy run worth splitting for
constexpr int64_t kMinSplitBytes = 32ll << 20;  // smaller problems: one piece
constexpr int kMaxPieces = 64;
constexpr size_t kFlagBytes = 256;  // per-piece "C piece arrived" flags, after the piece workspaces

// Page-locked constants the flags are copied from: kMaxPieces zeros, then kMaxPieces ones.
// The flags are written by the copy engine, in order behind the C uploads on the h2d
// stream: a kernel launch (cudaMemsetAsync, fill) could not get an SM while the pieces'
// persistent kernels, spinning on those flags, occupy all of them.
const int32_t *pinned_flag_values() {
  static std::once_flag once;
  static int32_t *v = nullptr;
  std::call_once(once, [] {
    if (cudaHostAlloc(reinterpret_cast<void **>(&v), 2 * kMaxPieces * sizeof(int32_t), cudaHostAllocPortable) !=
        cudaSuccess) {
      v = nullptr;
      return;
    }
    for (int i = 0; i < 2 * kMaxPieces; ++i) v[i] = i >= kMaxPieces;
  });
  return v;
}

// One tensor's labels (row bundle + column bundle).
struct TensorLabels {
  int n = 0;
  int64_t ext[2 * STC_MAX_LABELS], str[2 * STC_MAX_LABELS];
  int64_t base = 0;
  void add(const stc_bundle &b) {
    for (int d = 0; d < b.nlab; ++d) {
      ext[n] = b.ext[d];
      str[n] = b.str[d];
      ++n;
    }
  }
  int64_t elems() const {
    int64_t e = 1;
    for (int d = 0; d < n; ++d) e *= ext[d];
    return e;
  }
  // [lo, hi): the storage the tensor's elements occupy (strides of either sign; the
  // reference's DenseTensor allows negative strides, tensor.py:43-97)
  int64_t lo() const {
    int64_t l = base;
    for (int d = 0; d < n; ++d)
      if (str[d] < 0) l += (ext[d] - 1) * str[d];
    return l;
  }
  int64_t hi() const {
    int64_t h = base;
    for (int d = 0; d < n; ++d)
      if (str[d] > 0) h += (ext[d] - 1) * str[d];
    return elems() ? h + 1 : lo();
  }
  // strides a permutation of a dense row-major layout: the elements fill [base, base + elems)
  bool compact() const {
    std::vector<std::pair<int64_t, int64_t>> ls;
    for (int d = 0; d < n; ++d)
      if (ext[d] > 1) ls.push_back({str[d], ext[d]});
    std::sort(ls.begin(), ls.end());
    int64_t run = 1;
    for (auto &l : ls) {
      if (l.first != run) return false;
      run *= l.second;
    }
    return true;
  }
};

TensorLabels labels_of(const stc_bundle &r, const stc_bundle &c, int64_t base) {
  TensorLabels t;
  t.add(r);
  t.add(c);
  t.base = base;
  return t;
}

// A grid of pieces: label `la` of the I bundle (A rows and C rows) cut into `sa`
// equal ranges and label `lb` of the J bundle (B columns and C columns) into `sb`;
// piece s = r * sb + c holds I range r and J range c.  sa = 1 or sb = 1 is the 1-D
// split of round 1 (side / lab / pieces describe it for stc_host_plan).
struct Split {
  int la = 0, sa = 1, lb = 0, sb = 1;
  int side = 0, lab = 0, pieces = 1;  // 1-D view: the cut side (0: I, 1: J), its label, sa * sb
  int64_t run = 0;                    // shortest copy run, bytes
};

int64_t bundle_elems(const stc_bundle &b) {
  int64_t n = 1;
  for (int d = 0; d < b.nlab; ++d) n *= b.ext[d];
  return n;
}

Split one_d(int side, int lab, int S, int64_t run) {
  Split sp;
  sp.side = side;
  sp.lab = lab;
  sp.pieces = S;
  sp.run = run;
  if (side == 0) {
    sp.la = lab;
    sp.sa = S;
  } else {
    sp.lb = lab;
    sp.sb = S;
  }
  return sp;
}

// The best cut of one side into `want` (or fewer, halving) pieces: the label with the
// longest copy runs in both tensors it touches; false if none qualifies.
bool best_cut(const stc_problem &p, int side, int want, bool forced, int &lab, int &S, int64_t &run) {
  const stc_bundle &ob = side == 0 ? p.a_row : p.b_col;  // the operand's split bundle
  const stc_bundle &cb = side == 0 ? p.c_row : p.c_col;
  const int64_t quad = int64_t(1) << p.level;
  const int64_t blen = bundle_elems(cb);
  bool found = false;
  for (int l = 0; l < cb.nlab; ++l) {
    for (int n = want; n >= 2; n /= 2) {
      if (cb.ext[l] % n) continue;
      // each piece keeps at least two 128-wide tiles per quadrant, and copy runs
      // are long enough for full PCIe rate (forced counts: only divisibility)
      if (!forced && blen / n < quad * 256) continue;
      const int64_t r = 8 * (cb.ext[l] / n) * std::min(ob.str[l], cb.str[l]);
      if (!forced && r < kMinRunBytes) continue;
      if (!found || n > S || (n == S && r > run)) {
        lab = l;
        S = n;
        run = r;
        found = true;
      }
      break;
    }
  }
  return found;
}

Split choose_split(const stc_problem &p) {
  Split best;
  const TensorLabels A = labels_of(p.a_row, p.a_col, p.a_base), B = labels_of(p.b_row, p.b_col, p.b_base),
                     C = labels_of(p.c_row, p.c_col, p.c_base);
  const int64_t bytes = 8 * (A.elems() + B.elems() + 2 * C.elems());
  if (!C.compact()) return best;
  // I x J grid (STC_HOST_GRID=SAxSB forces it, "1" disables): for problems of 16 GB and
  // more a 1-D cut must upload a whole operand before the first piece can start (cfg5:
  // 8.6 GB, 0.17 s); a 4 x 8 grid starts after a quarter of A and an eighth of B (0.06 s).
  // With the pieces sharing their operand slots (Share) the finer grid costs no extra
  // pre-summing: cfg5 e2e 4 x 4 1637 ms, 4 x 8 1609 ms (8 x 8: 1877 ms, pieces too thin).
  // From 12 GB on, J cut in 8 when that leaves pieces at least 4096 wide, else in 4 (the
  // cfg5 shard of 4 GPUs, 32768 x 8192: 4 x 4 435 ms, 4 x 8 452 ms, 1-D 482 ms)
  const char *genv = getenv("STC_HOST_GRID");
  int ga = 0, gb = 0;
  if (genv && sscanf(genv, "%dx%d", &ga, &gb) != 2) ga = gb = 0;
  const char *env = getenv("STC_HOST_PIECES");
  if (!env && (ga > 0 || (!genv && bytes >= (12ll << 30))) && A.compact() && B.compact()) {
    const bool forced = ga > 0;
    int la = 0, lb = 0, sa = 0, sb = 0;
    int64_t ra = 0, rb = 0;
    const int jb = bundle_elems(p.c_col) / 8 >= 4096 ? 8 : 4;
    if (best_cut(p, 0, forced ? ga : 4, forced, la, sa, ra) && best_cut(p, 1, forced ? gb : jb, forced, lb, sb, rb) &&
        sa * sb <= kMaxPieces && (forced || (sa >= 2 && sb >= 2))) {
      best.la = la;
      best.sa = sa;
      best.lb = lb;
      best.sb = sb;
      best.side = 0;
      best.lab = la;
      best.pieces = sa * sb;
      best.run = std::min(ra, rb);
      return best;
    }
  }
  // 1-D: 4 pieces; 8 for problems of 4 GB and more (the first piece after an eighth of the
  // cut operand; a shorter tail: the last C piece's download).  The cfg5 shard of 8 GPUs
  // (32768 x 4096, 11 GB): 8 pieces 240 ms, 4 pieces 262 ms
  const int want = env ? std::max(1, std::min(kMaxPieces, atoi(env))) : (bytes >= (4ll << 30) ? 8 : 4);
  if (want <= 1 || (!env && bytes < kMinSplitBytes)) return best;
  for (int side = 0; side < 2; ++side) {
    if (!(side == 0 ? A : B).compact()) continue;
    int l = 0, S = 0;
    int64_t run = 0;
    if (!best_cut(p, side, want, env != nullptr, l, S, run)) continue;
    const bool better = S > best.pieces || (S == best.pieces && run > best.run);
    if (better) best = one_d(side, l, S, run);
  }
  return best;
}

// The piece's I range [i0, i0 + ni) of label la and J range [j0, j0 + nj) of label lb:
// those labels' extents in the tensors they index reduced, the bases moved.
stc_problem piece_problem(const stc_problem &p, const Split &sp, int64_t i0, int64_t ni, int64_t j0, int64_t nj) {
  stc_problem q = p;
  if (sp.sa > 1) {
    q.a_row.ext[sp.la] = ni;
    q.c_row.ext[sp.la] = ni;
    q.a_base += i0 * p.a_row.str[sp.la];
    q.c_base += i0 * p.c_row.str[sp.la];
  }
  if (sp.sb > 1) {
    q.b_col.ext[sp.lb] = nj;
    q.c_col.ext[sp.lb] = nj;
    q.b_base += j0 * p.b_col.str[sp.lb];
    q.c_base += j0 * p.c_col.str[sp.lb];
  }
  return q;
}

// Ranges of piece s: I range r = s / sb of label la, J range c = s % sb of label lb.
struct PieceRange {
  int64_t i0 = 0, ni = 1, j0 = 0, nj = 1;
};
PieceRange piece_range(const stc_problem &p, const Split &sp, int s) {
  PieceRange pr;
  const int r = s / sp.sb, c = s % sp.sb;
  if (sp.sa > 1) {
    const int64_t e = p.c_row.ext[sp.la];
    pr.i0 = e * r / sp.sa;
    pr.ni = e * (r + 1) / sp.sa - pr.i0;
  }
  if (sp.sb > 1) {
    const int64_t e = p.c_col.ext[sp.lb];
    pr.j0 = e * c / sp.sb;
    pr.nj = e * (c + 1) / sp.sb - pr.j0;
  }
  return pr;
}

// Copy of the elements of compact tensor t with one label (stride lstr,
// extent lext) restricted to [r0, r0 + len): rows of len * lstr elements at
// pitch lext * lstr.
cudaError_t copy_piece(double *dst, const double *src, const TensorLabels &t, int64_t lstr, int64_t lext,
                       int64_t r0, int64_t len, cudaMemcpyKind kind, cudaStream_t s) {
  const int64_t pitch = lext * lstr, rows = t.elems() / pitch;
  const int64_t off = t.base + r0 * lstr;
  return cudaMemcpy2DAsync(dst + off, pitch * 8, src + off, pitch * 8, len * lstr * 8, rows, kind, s);
}

// The elements of compact tensor t with label X (stride xs, extent xe) restricted to
// [x0, x0 + xn) and label Y (stride ys, extent ye) to [y0, y0 + yn): for every index of
// the outer of the two (the larger stride) one 2-D copy of the inner one's restriction.
cudaError_t copy_block(double *dst, const double *src, const TensorLabels &t, int64_t xs, int64_t xe, int64_t x0,
                       int64_t xn, int64_t ys, int64_t ye, int64_t y0, int64_t yn, cudaMemcpyKind kind,
                       cudaStream_t s) {
  if (xs < ys) {
    std::swap(xs, ys);
    std::swap(xe, ye);
    std::swap(x0, y0);
    std::swap(xn, yn);
  }
  // outer label x (stride xs), inner y: within one x index, rows of ye * ys elements;
  // the labels outside x (strides >= xs * xe, compact) are `outer` blocks of xs * xe
  const int64_t pitch = ye * ys, rows = xs / pitch, outer = t.elems() / (xs * xe);
  for (int64_t o = 0; o < outer; ++o)
    for (int64_t v = x0; v < x0 + xn; ++v) {
      const int64_t off = t.base + o * xs * xe + v * xs + y0 * ys;
      cudaError_t e = cudaMemcpy2DAsync(dst + off, pitch * 8, src + off, pitch * 8, yn * ys * 8, rows, kind, s);
      if (e != cudaSuccess) return e;
    }
  return cudaSuccess;
}

cudaError_t copy_span(double *dst, const double *src, const TensorLabels &t, cudaMemcpyKind kind, cudaStream_t s) {
  const int64_t lo = t.lo(), n = t.hi() - lo;
  if (n <= 0) return cudaSuccess;
  return cudaMemcpyAsync(dst + lo, src + lo, n * 8, kind, s);
}

struct HostStreams {
  bool init = false;
  cudaStream_t h2d = nullptr, d2h = nullptr, comp[2] = {nullptr, nullptr};
};
HostStreams g_hs[64];
std::mutex g_hs_mu;

int host_streams(HostStreams *&hs) {
  int dev = 0;
  HCU(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_hs_mu);
  hs = &g_hs[dev & 63];
  if (!hs->init) {
    HCU(cudaStreamCreateWithFlags(&hs->h2d, cudaStreamNonBlocking), "cudaStreamCreate");
    HCU(cudaStreamCreateWithFlags(&hs->d2h, cudaStreamNonBlocking), "cudaStreamCreate");
    for (auto &c : hs->comp) HCU(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking), "cudaStreamCreate");
    hs->init = true;
  }
  return STC_OK;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// An error after the first enqueue returns while copies and kernels may still be
// queued on the library's streams, reading and writing the caller's buffers: wait
// for them before handing control (and the buffers) back.
struct DrainOnError {
  HostStreams *hs = nullptr;
  bool armed = true;
  ~DrainOnError() {
    if (!armed || !hs) return;
    for (cudaStream_t s : {hs->h2d, hs->d2h, hs->comp[0], hs->comp[1]})
      if (s) cudaStreamSynchronize(s);
    cudaGetLastError();
  }
};

// The first cell of a grid split along one label of the P bundle: its runs (k parts, one
// after the other on one stream, adding into the same C block) start after a part of
// its A and B blocks arrived (cfg5, 4 x 8: 15 ms instead of 53 ms of PCIe before the first
// DMMA).  The label: the P label with the largest stride in A that the parts divide
// (long copy runs).  STC_HOST_KSPLIT=n forces n parts, 0 disables.
struct KSplit {
  bool on = false;
  int lk = 0;                  // the P bundle label
  int parts = 0;               // its ranges (STC_HOST_KSPLIT=n: n parts, 0 disables; default 2)
  int64_t k0[4] = {}, kn[4] = {};
};

KSplit plan_ksplit(const stc_problem &p, const Split &sp) {
  KSplit ks;
  if (sp.sa < 2 || sp.sb < 2) return ks;
  // 4 parts (cfg5: the first DMMA after 15 ms; 2 parts 1568 ms, 4 parts 1564 ms per call), else 2
  int n = 4;
  const char *env = getenv("STC_HOST_KSPLIT");
  if (env) n = std::max(0, std::min(4, atoi(env)));
  int64_t k = 1;
  for (int d = 0; d < p.a_col.nlab; ++d) k *= p.a_col.ext[d];
  int best = -1;
  for (; n >= 2; n = env ? 0 : n / 2) {
    best = -1;
    for (int d = 0; d < p.a_col.nlab; ++d)
      if (p.a_col.ext[d] >= n && p.a_col.ext[d] % n == 0 && (best < 0 || p.a_col.str[d] > p.a_col.str[best]))
        best = d;
    // parts of at least two 16-deep chunks per quadrant
    if (best >= 0 && k / n >= ((int64_t)2 << p.level) * 16) break;
  }
  if (n < 2 || best < 0) return ks;
  ks.on = true;
  ks.lk = best;
  ks.parts = n;
  const int64_t e = p.a_col.ext[best];
  for (int i = 0; i < n; ++i) {
    ks.k0[i] = e * i / n;
    ks.kn[i] = e * (i + 1) / n - ks.k0[i];
  }
  return ks;
}

// Half kh of a cell's problem: the split P label's extent in A and B halved, bases moved.
stc_problem half_problem(const stc_problem &cell, const KSplit &ks, int kh) {
  stc_problem q = cell;
  q.a_col.ext[ks.lk] = ks.kn[kh];
  q.b_row.ext[ks.lk] = ks.kn[kh];
  q.a_base += ks.k0[kh] * cell.a_col.str[ks.lk];
  q.b_base += ks.k0[kh] * cell.b_row.str[ks.lk];
  return q;
}

// Workspace of one piece slot: the largest over the pieces (their plans differ in the
// base offsets, which can change the path -- e.g. whether a view is a TMA box -- and
// with it the workspace).
int piece_workspace(const stc_problem &p, const Split &sp, const KSplit &ks, size_t &per_slot) {
  size_t most = 256;
  for (int s = 0; s < sp.pieces; ++s) {
    const PieceRange pr = piece_range(p, sp, s);
    stc_problem q = sp.pieces > 1 ? piece_problem(p, sp, pr.i0, pr.ni, pr.j0, pr.nj) : p;
    size_t b = 0;
    if (int rc = stc_workspace_size(&q, &b)) return rc;
    most = std::max(most, b);
    if (s == 0 && ks.on)
      for (int kh = 0; kh < ks.parts; ++kh) {
        const stc_problem h = half_problem(q, ks, kh);
        if (int rc = stc_workspace_size(&h, &b)) return rc;
        most = std::max(most, b);
      }
  }
  per_slot = align256(most);
  return STC_OK;
}

// Operand slots shared between the pieces of a grid (SlotOverride): the pre-summed A
// slots of I range r are formed once, by piece (r, 0), into one of two alternating
// buffers, and read by the pieces (r, 1..); the B slots of J range c once, by piece
// (0, c), into buffer c.  Without it every piece re-forms both (cfg5, 4 x 4 grid: 43 ms
// of pre-summing instead of 11).  Needs a uniform grid whose pieces pre-sum both sides
// in one batch; STC_HOST_SHARE=0 disables.
// A 1-D split shares the operand all its pieces use whole: B for a cut of the I bundle,
// A for a cut of the J bundle.
struct Share {
  bool on = false, a = false, b = false;  // any / the A side / the B side shared
  size_t a_bytes = 0, b_bytes = 0;        // one A / one B slot buffer (256-aligned)
  size_t bytes(const Split &sp) const {
    return (a ? 2 * a_bytes : 0) + (b ? (size_t)sp.sb * b_bytes : 0);
  }
};

Share plan_share(const stc_problem &p, const Split &sp) {
  Share sh;
  if (sp.pieces < 2) return sh;
  if (const char *e = getenv("STC_HOST_SHARE"))
    if (atoi(e) == 0) return sh;
  size_t a0 = 0, b0 = 0;
  for (int s = 0; s < sp.pieces; ++s) {
    const PieceRange pr = piece_range(p, sp, s);
    const stc_problem q = piece_problem(p, sp, pr.i0, pr.ni, pr.j0, pr.nj);
    size_t a = 0, b = 0;
    if (!plan_slot_bytes(&q, a, b)) return sh;
    if (s == 0) {
      a0 = a;
      b0 = b;
    } else if (a != a0 || b != b0) {
      return sh;  // pieces of different shapes: their slots differ
    }
  }
  if (a0 == 0 || b0 == 0) return sh;
  sh.a = sp.sb >= 2;  // A row blocks are reused along the J cut
  sh.b = sp.sa >= 2;  // B column blocks along the I cut
  sh.on = sh.a || sh.b;
  sh.a_bytes = align256(a0);
  sh.b_bytes = align256(b0);
  return sh;
}

// RAII set of events, destroyed after enqueue (the runtime releases them when
// the work they mark completes).
struct Events {
  std::vector<cudaEvent_t> ev;
  ~Events() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
  cudaError_t make(cudaEvent_t &e) {
    cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (r == cudaSuccess) ev.push_back(e);
    return r;
  }
};

// cuStreamWaitValue32 (driver API stream memory operation): the download stream
// waits on the device-side item counter of a piece (gated mode).
}  // namespace

extern "C" {

int stc_host_grid(const stc_problem *p, int32_t *i_label, int32_t *i_pieces, int32_t *j_label, int32_t *j_pieces) {
  if (!p) return herr(STC_EINVAL, "null problem");
  const Split sp = choose_split(*p);
  if (i_label) *i_label = sp.la;
  if (i_pieces) *i_pieces = sp.sa;
  if (j_label) *j_label = sp.lb;
  if (j_pieces) *j_pieces = sp.sb;
  return STC_OK;
}

int stc_host_plan(const stc_problem *p, int32_t *side, int32_t *label, int32_t *pieces) {
  if (!p) return herr(STC_EINVAL, "null problem");
  const Split sp = choose_split(*p);
  if (side) *side = sp.side;
  if (label) *label = sp.lab;
  if (pieces) *pieces = sp.pieces;
  return STC_OK;
}

int stc_host_workspace_size(const stc_problem *p, size_t *bytes) {
  if (!p) return herr(STC_EINVAL, "null problem");
  const Split sp = choose_split(*p);
  size_t per = 0;
  if (int rc = piece_workspace(*p, sp, plan_ksplit(*p, sp), per)) return rc;
  size_t need = per * (sp.pieces > 1 ? 2 : 1) + kFlagBytes + plan_share(*p, sp).bytes(sp);
  if (bytes) *bytes = need;
  return STC_OK;
}

int stc_contract_host(const stc_problem *p, const double *hA, const double *hB, double *hC, double *dA, double *dB,
                      double *dC, void *workspace, size_t workspace_bytes, void *stream, stc_stats *stats) {
  if (!p) return herr(STC_EINVAL, "null problem");
  if (!hA || !hB || !hC || !dA || !dB || !dC) return herr(STC_EINVAL, "null operand pointer");
  const Split sp = choose_split(*p);
  const KSplit ks = plan_ksplit(*p, sp);
  size_t per = 0;
  if (int rc = piece_workspace(*p, sp, ks, per)) return rc;
  const int slots = sp.pieces > 1 ? 2 : 1;
  const Share share = plan_share(*p, sp);
  const size_t need = per * slots + kFlagBytes + share.bytes(sp);
  if (!workspace || workspace_bytes < need)
    return herr(STC_EWORKSPACE, "workspace too small: need %zu bytes, got %zu", need, workspace_bytes);
  if (reinterpret_cast<uintptr_t>(workspace) & 255) return herr(STC_EINVAL, "workspace must be 256-byte aligned");
  // the cells: an I range x a J range each (the grid of choose_split); the runs: one
  // contraction per cell, or -- the first cell k-split (KSplit) -- two in k order
  std::vector<PieceRange> ranges;
  std::vector<stc_problem> cells;
  for (int s = 0; s < sp.pieces; ++s) {
    const PieceRange pr = piece_range(*p, sp, s);
    cells.push_back(sp.pieces > 1 ? piece_problem(*p, sp, pr.i0, pr.ni, pr.j0, pr.nj) : *p);
    ranges.push_back(pr);
  }
  struct Run {
    int cell, kh;  // kh: -1 the whole k range, else the part of KSplit
    stc_problem prob;
  };
  std::vector<Run> runs;
  for (int s = 0; s < sp.pieces; ++s) {
    if (s == 0 && ks.on) {
      for (int kh = 0; kh < ks.parts; ++kh) runs.push_back({0, kh, half_problem(cells[0], ks, kh)});
    } else {
      runs.push_back({s, -1, cells[s]});
    }
  }
  const int nruns = (int)runs.size();
  HostStreams *hs = nullptr;
  if (int rc = host_streams(hs)) return rc;
  DrainOnError drain;
  drain.hs = hs;
  // the per-call hooks belong to device-operand calls
  stc_set_c_ready(nullptr);
  stc_set_kernel_events(nullptr, nullptr);

  const TensorLabels A = labels_of(p->a_row, p->a_col, p->a_base), B = labels_of(p->b_row, p->b_col, p->b_base),
                     C = labels_of(p->c_row, p->c_col, p->c_base);
  cudaStream_t us = reinterpret_cast<cudaStream_t>(stream);
  Events E;
  cudaEvent_t start, end;
  HCU(E.make(start), "cudaEventCreate");
  HCU(E.make(end), "cudaEventCreate");
  HCU(cudaEventRecord(start, us), "cudaEventRecord");
  // STC_HOST_TRACE=1: timing events per run (inputs in, compute start / end, C out), printed to stderr
  const bool trace = getenv("STC_HOST_TRACE") != nullptr;
  std::vector<cudaEvent_t> tr(trace ? 1 + 4 * nruns : 0);
  for (auto &e : tr) HCU(cudaEventCreate(&e), "cudaEventCreate");
  if (trace) HCU(cudaEventRecord(tr[0], us), "cudaEventRecord");
  for (cudaStream_t s : {hs->h2d, hs->d2h, hs->comp[0], hs->comp[1]})
    HCU(cudaStreamWaitEvent(s, start, 0), "cudaStreamWaitEvent");

  // uploads: the operand all pieces share, then (operand piece, C piece, flag) per piece.
  // A run's kernels start once its operands are in (event opin) and wait on the
  // device for its cell's flag before their first access to C (stc_set_c_ready), so
  // the C upload overlaps the piece's first MMAs.
  const int32_t *pf = pinned_flag_values();
  if (!pf) return herr(STC_ECUDA, "cudaHostAlloc failed for the piece flags");
  int32_t *flags = reinterpret_cast<int32_t *>(reinterpret_cast<char *>(workspace) + per * slots);
  HCU(cudaMemcpyAsync(flags, pf, sp.pieces * sizeof(int32_t), cudaMemcpyHostToDevice, hs->h2d),
      "cudaMemcpyAsync(flags)");
  std::vector<cudaEvent_t> opin(nruns), done(nruns);
  std::vector<int> first_run(sp.pieces, -1), last_run(sp.pieces, -1);  // of each cell
  for (int k = 0; k < nruns; ++k) {
    if (first_run[runs[k].cell] < 0) first_run[runs[k].cell] = k;
    last_run[runs[k].cell] = k;
  }
  auto c_arrived = [&](int cell) -> int {
    HCU(cudaMemcpyAsync(flags + cell, pf + kMaxPieces, sizeof(int32_t), cudaMemcpyHostToDevice, hs->h2d),
        "cudaMemcpyAsync(flag)");
    if (trace) HCU(cudaEventRecord(tr[1 + 4 * first_run[cell]], hs->h2d), "cudaEventRecord");
    return STC_OK;
  };
  // A's I range r (all of A when the I bundle is not cut), B's J range c, C's block;
  // kh >= 0: only the k half kh of them (the k-split first cell)
  auto copy_a = [&](int r, int kh) -> cudaError_t {
    const PieceRange &pr = ranges[r * sp.sb];
    if (kh >= 0)
      return copy_block(dA, hA, A, p->a_row.str[sp.la], p->a_row.ext[sp.la], pr.i0, pr.ni, p->a_col.str[ks.lk],
                        p->a_col.ext[ks.lk], ks.k0[kh], ks.kn[kh], cudaMemcpyHostToDevice, hs->h2d);
    if (sp.sa == 1) return copy_span(dA, hA, A, cudaMemcpyHostToDevice, hs->h2d);
    return copy_piece(dA, hA, A, p->a_row.str[sp.la], p->a_row.ext[sp.la], pr.i0, pr.ni, cudaMemcpyHostToDevice,
                      hs->h2d);
  };
  auto copy_b = [&](int c, int kh) -> cudaError_t {
    const PieceRange &pr = ranges[c];
    if (kh >= 0)
      return copy_block(dB, hB, B, p->b_row.str[ks.lk], p->b_row.ext[ks.lk], ks.k0[kh], ks.kn[kh],
                        p->b_col.str[sp.lb], p->b_col.ext[sp.lb], pr.j0, pr.nj, cudaMemcpyHostToDevice, hs->h2d);
    if (sp.sb == 1) return copy_span(dB, hB, B, cudaMemcpyHostToDevice, hs->h2d);
    return copy_piece(dB, hB, B, p->b_col.str[sp.lb], p->b_col.ext[sp.lb], pr.j0, pr.nj, cudaMemcpyHostToDevice,
                      hs->h2d);
  };
  auto copy_c = [&](double *dst, const double *src, int cell, cudaMemcpyKind kind, cudaStream_t st) -> cudaError_t {
    const PieceRange &pr = ranges[cell];
    if (sp.sa > 1 && sp.sb > 1)
      return copy_block(dst, src, C, p->c_row.str[sp.la], p->c_row.ext[sp.la], pr.i0, pr.ni, p->c_col.str[sp.lb],
                        p->c_col.ext[sp.lb], pr.j0, pr.nj, kind, st);
    if (sp.sa > 1) return copy_piece(dst, src, C, p->c_row.str[sp.la], p->c_row.ext[sp.la], pr.i0, pr.ni, kind, st);
    if (sp.sb > 1) return copy_piece(dst, src, C, p->c_col.str[sp.lb], p->c_col.ext[sp.lb], pr.j0, pr.nj, kind, st);
    return copy_span(dst, src, C, kind, st);
  };
  // uploads in run order: A's range r, B's range c (first row of the grid only), then the
  // cell's C block and its arrival flag; the k-split first cell: its halves' A and B
  // blocks one after the other (the first half's run starts after half the data)
  for (int k = 0; k < nruns; ++k) {
    const Run &ru = runs[k];
    const int r = ru.cell / sp.sb, c = ru.cell % sp.sb;
    if (ru.kh >= 0) {
      HCU(copy_a(r, ru.kh), "cudaMemcpyAsync(A piece)");
      HCU(copy_b(c, ru.kh), "cudaMemcpyAsync(B piece)");
    } else {
      if (c == 0) HCU(copy_a(r, -1), "cudaMemcpyAsync(A piece)");
      if (r == 0) HCU(copy_b(c, -1), "cudaMemcpyAsync(B piece)");
    }
    HCU(E.make(opin[k]), "cudaEventCreate");
    HCU(cudaEventRecord(opin[k], hs->h2d), "cudaEventRecord");
    if (k == first_run[ru.cell]) {
      HCU(copy_c(dC, hC, ru.cell, cudaMemcpyHostToDevice, hs->h2d), "cudaMemcpyAsync(C piece)");
      if (int rc = c_arrived(ru.cell)) return rc;
    }
  }
  // plan every run before any of them is launched (the uploads above only fill the
  // caller's device buffers; on an error they are drained before returning)
  for (int k = 0; k < nruns; ++k) {
    size_t nb = 0;
    if (int rc = stc_workspace_size(&runs[k].prob, &nb)) {
      cudaStreamSynchronize(hs->h2d);
      return rc;
    }
  }
  // download of a cell's C once its last run finished
  auto download = [&](int k) -> int {
    const int cell = runs[k].cell;
    HCU(cudaStreamWaitEvent(hs->d2h, done[k], 0), "cudaStreamWaitEvent");
    HCU(copy_c(hC, dC, cell, cudaMemcpyDeviceToHost, hs->d2h), "cudaMemcpyAsync(C piece)");
    if (trace) HCU(cudaEventRecord(tr[4 + 4 * k], hs->d2h), "cudaEventRecord");
    return STC_OK;
  };
  // page-locked C: each download is enqueued right behind its piece (asynchronous);
  // pageable C: after all pieces (such copies block the host until they ran)
  cudaPointerAttributes pa{};
  const bool locked = cudaPointerGetAttributes(&pa, hC) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  cudaGetLastError();  // a failed query leaves an error code behind
  // pieces on alternating compute streams (workspace slot = stream), so piece s+1's
  // CTAs fill the SMs of piece s's last wave -- unless the pieces run through dense M
  // slots (stc_contract's dense-M ABC mode, AB, Naive): their accumulate kernels would
  // then wait behind the next piece's persistent kernel, and one stream is faster.
  // The runs of one cell (k halves) update the same C block: the later waits for the
  // earlier.
  const bool alternate = plan_ticketed(&cells[0]);
  stc_stats total{};
  char *ws = reinterpret_cast<char *>(workspace);
  char *shared = ws + per * slots + kFlagBytes;  // A slot buffers [2], then B slot buffers [sb]
  // the run forming the shared slots of A range r / B range c: the first whole-k run of
  // the row / column (KSplit's halves form their own)
  std::vector<int> form_a(sp.sa, -1), form_b(sp.sb, -1);
  for (int k = 0; k < nruns; ++k) {
    if (runs[k].kh >= 0) continue;
    const int r = runs[k].cell / sp.sb, c = runs[k].cell % sp.sb;
    if (form_a[r] < 0) form_a[r] = k;
    if (form_b[c] < 0) form_b[c] = k;
  }
  std::vector<cudaEvent_t> formed(nruns, nullptr);
  for (int k = 0; k < nruns; ++k) {
    const Run &ru = runs[k];
    const int r = ru.cell / sp.sb, c = ru.cell % sp.sb;
    cudaStream_t cs = hs->comp[alternate ? k % slots : 0];
    HCU(cudaStreamWaitEvent(cs, opin[k], 0), "cudaStreamWaitEvent");
    if (k > first_run[ru.cell]) HCU(cudaStreamWaitEvent(cs, done[k - 1], 0), "cudaStreamWaitEvent");
    if (trace) HCU(cudaEventRecord(tr[2 + 4 * k], cs), "cudaEventRecord");
    SlotOverride ovr;
    const bool shares = share.on && ru.kh < 0 && form_a[r] >= 0 && form_b[c] >= 0;
    if (shares) {
      // a side not shared keeps its slots in the piece's own workspace (pa / pb null)
      char *sb_base = shared + (share.a ? 2 * share.a_bytes : 0);
      ovr.pa = share.a ? reinterpret_cast<double *>(shared + (r % 2) * share.a_bytes) : nullptr;
      ovr.pb = share.b ? reinterpret_cast<double *>(sb_base + c * share.b_bytes) : nullptr;
      ovr.skip_a = share.a && k != form_a[r];
      ovr.skip_b = share.b && k != form_b[c];
      if (ovr.skip_a) HCU(cudaStreamWaitEvent(cs, formed[form_a[r]], 0), "cudaStreamWaitEvent");
      if (ovr.skip_b) HCU(cudaStreamWaitEvent(cs, formed[form_b[c]], 0), "cudaStreamWaitEvent");
      if (share.a && !ovr.skip_a && r >= 2)  // A buffer r % 2: the runs of I range r - 2 are done reading it
        for (int j = 0; j < nruns; ++j)
          if (runs[j].cell / sp.sb == r - 2) HCU(cudaStreamWaitEvent(cs, done[j], 0), "cudaStreamWaitEvent");
      if ((share.a && !ovr.skip_a) || (share.b && !ovr.skip_b)) {
        HCU(E.make(formed[k]), "cudaEventCreate");
        ovr.after_presum = formed[k];
      }
    }
    stc_stats st{};
    stc_set_c_ready(flags + ru.cell);
    if (shares) set_slot_override(&ovr);
    if (int rc = stc_contract(&ru.prob, dA, dB, dC, ws + (k % slots) * per, per, cs, &st)) {
      stc_set_c_ready(nullptr);
      set_slot_override(nullptr);
      return rc;
    }
    HCU(E.make(done[k]), "cudaEventCreate");
    HCU(cudaEventRecord(done[k], cs), "cudaEventRecord");
    if (trace) HCU(cudaEventRecord(tr[3 + 4 * k], cs), "cudaEventRecord");
    total.total_flops += st.total_flops;
    total.fast_blocks += st.fast_blocks;
    total.slow_blocks += st.slow_blocks;
    total.fast_updates += st.fast_updates;
    total.slow_updates += st.slow_updates;
    total.leaf_multiplies = std::max(total.leaf_multiplies, st.leaf_multiplies);
    total.work_items += st.work_items;
    total.kernel_launches += st.kernel_launches;
    if (locked && k == last_run[ru.cell])
      if (int rc = download(k)) return rc;
  }
  if (!locked)
    for (int k = 0; k < nruns; ++k)
      if (k == last_run[runs[k].cell])
        if (int rc = download(k)) return rc;
  HCU(cudaEventRecord(end, hs->d2h), "cudaEventRecord");
  if (trace) {
    cudaEventSynchronize(end);
    float t = 0;
    fprintf(stderr, "[stc host] runs=%d (I label %d x %d, J label %d x %d, k-split first cell %d):", nruns, sp.la,
            sp.sa, sp.lb, sp.sb, ks.on ? 1 : 0);
    for (int k = 0; k < nruns; ++k) {
      fprintf(stderr, " |%d", k);
      for (int j = 0; j < 4; ++j) {
        const int idx = j == 0 ? first_run[runs[k].cell] : j == 3 ? last_run[runs[k].cell] : k;
        cudaEventElapsedTime(&t, tr[0], tr[1 + 4 * idx + j]);
        fprintf(stderr, " %.2f", t);
      }
    }
    fprintf(stderr, "  (C in, kstart, kend, out ms)\n");
    for (cudaEvent_t e : tr) cudaEventDestroy(e);
  }
  HCU(cudaStreamWaitEvent(us, end, 0), "cudaStreamWaitEvent");
  drain.armed = false;
  total.pieces = nruns;
  if (stats) *stats = total;
  return STC_OK;
}

int stc_sharded_workspace_size(const stc_problem *p, int ngpu, int label, size_t *bytes) {
  if (!p || ngpu < 1) return herr(STC_EINVAL, "null problem or no devices");
  size_t most = 256;
  int32_t lab = label;
  for (int g = 0; g < ngpu; ++g) {
    stc_problem q;
    if (int rc = stc_shard_problem(p, ngpu, g, lab, &q, nullptr, nullptr, &lab)) return rc;
    size_t b = 0;
    if (int rc = stc_workspace_size(&q, &b)) return rc;
    most = std::max(most, b);
  }
  if (bytes) *bytes = most;
  return STC_OK;
}

int stc_contract_sharded(const stc_problem *p, int ngpu, const int *devices, int label, const double *const *A,
                         const double *const *B, double *const *C, void *const *workspace,
                         const size_t *workspace_bytes, void *const *streams, int gather, stc_stats *stats) {
  if (!p || ngpu < 1 || !devices || !A || !B || !C || !workspace || !workspace_bytes || !streams)
    return herr(STC_EINVAL, "null argument or no devices");
  const TensorLabels Ct = labels_of(p->c_row, p->c_col, p->c_base);
  if (gather && ngpu > 1 && !Ct.compact()) return herr(STC_EINVAL, "gather needs a compact C (dense storage)");
  int cur = 0;
  HCU(cudaGetDevice(&cur), "cudaGetDevice");
  struct Restore {
    int dev;
    ~Restore() { cudaSetDevice(dev); }
  } restore{cur};
  // the shards (the label fixed by shard 0's choice)
  std::vector<stc_problem> q(ngpu);
  std::vector<int64_t> s0(ngpu), s1(ngpu);
  int32_t lab = label;
  for (int g = 0; g < ngpu; ++g)
    if (int rc = stc_shard_problem(p, ngpu, g, lab, &q[g], &s0[g], &s1[g], &lab)) return rc;
  stc_set_c_ready(nullptr);
  stc_set_kernel_events(nullptr, nullptr);
  Events E;
  std::vector<cudaEvent_t> done(ngpu);
  stc_stats total{};
  for (int g = 0; g < ngpu; ++g) {
    HCU(cudaSetDevice(devices[g]), "cudaSetDevice");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(streams[g]);
    stc_stats st{};
    if (int rc = stc_contract(&q[g], A[g], B[g], C[g], workspace[g], workspace_bytes[g], s, &st)) return rc;
    HCU(E.make(done[g]), "cudaEventCreate");
    HCU(cudaEventRecord(done[g], s), "cudaEventRecord");
    total.total_flops += st.total_flops;
    total.fast_blocks += st.fast_blocks;
    total.slow_blocks += st.slow_blocks;
    total.fast_updates += st.fast_updates;
    total.slow_updates += st.slow_updates;
    total.leaf_multiplies = std::max(total.leaf_multiplies, st.leaf_multiplies);
    total.work_items += st.work_items;
    total.kernel_launches += st.kernel_launches;
  }
  if (gather && ngpu > 1) {
    // peer access where the devices differ (an already enabled pair is fine)
    for (int d = 0; d < ngpu; ++d)
      for (int g = 0; g < ngpu; ++g)
        if (devices[d] != devices[g]) {
          int ok = 0;
          if (cudaDeviceCanAccessPeer(&ok, devices[d], devices[g]) == cudaSuccess && ok) {
            cudaSetDevice(devices[d]);
            cudaDeviceEnablePeerAccess(devices[g], 0);
          }
          cudaGetLastError();
        }
    // device d's C gets shard g's block of C[g]: rows of the label's range at its pitch
    const int64_t lstr = p->c_col.str[lab], lext = p->c_col.ext[lab];
    for (int d = 0; d < ngpu; ++d) {
      HCU(cudaSetDevice(devices[d]), "cudaSetDevice");
      cudaStream_t s = reinterpret_cast<cudaStream_t>(streams[d]);
      for (int g = 0; g < ngpu; ++g) {
        if (g == d) continue;
        HCU(cudaStreamWaitEvent(s, done[g], 0), "cudaStreamWaitEvent");
        HCU(copy_piece(C[d], C[g], Ct, lstr, lext, s0[g], s1[g] - s0[g], cudaMemcpyDefault, s),
            "cudaMemcpy2DAsync(peer C block)");
      }
    }
  }
  total.pieces = ngpu;
  if (stats) *stats = total;
  return STC_OK;
}

}  // extern "C"
