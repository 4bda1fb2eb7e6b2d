// C ABI (include/cjt.h): plan upload, work-list construction, batched
// execution of the forward / inverse transform, and the reference
// backend-plugin entry points.
//
// Execution order (one stream, no host synchronisation inside cjt_execute):
//   forward (engine.py:153-186)
//     1. K1 recurrence contraction (split-K items)      -> partials
//     2. fixed-order partial reduction                   -> values[b][0..G]
//     3. per asymptotic block: chirp-z, summed over m    -> values += ...
//     4. Chebyshev analysis chirp-z                      -> out[b][0..N]
//   inverse (engine.py:189-227)
//     1. weighted Chebyshev synthesis chirp-z            -> wv[b][0..G]
//     2. per asymptotic block (degrees <= N only)        -> acc[b][0..N]
//     3. K2 recurrence contraction (degrees <= N only)   -> partials
//     4. fixed-order reduction, + acc, * 1/A_n           -> out[b][0..N]
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include "cjt_internal.cuh"

namespace cjt {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

}  // namespace cjt

using namespace cjt;

struct cjt_plan {
  int device = 0;
  int direction = 0;
  int m_terms = 0;
  int64_t n = 0, G = 0, nrows = 0;
  std::vector<void*> allocs;

  RecRowsDev rows{};
  RecTablesDev tab{};
  std::vector<int64_t> h_cut;
  int64_t* ck_off = nullptr;
  double2* ck = nullptr;
  int64_t ck_count = 0;
  int64_t rec_steps = 0;

  std::vector<ChirpZDev> blocks;
  ChirpZDev edge{};
  bool has_edge = false;
  double2* tw8192 = nullptr;
  double* scal = nullptr;
  int64_t scratch_elems_per_vec = 0;  // complex elements of multipass scratch per vector
  double fft_points = 0.0;

  // batch-dependent state (cjt_plan_reserve)
  int64_t reserved = 0;
  std::vector<void*> ws_allocs;
  FwdItem* fitems = nullptr;
  int64_t n_fitems = 0;
  int32_t* tile_slot0 = nullptr;
  int32_t* tile_nslot = nullptr;
  int64_t n_fslots = 0;
  // alpha = beta parity folding: P_n(-x) = (-1)^n P_n(x) on the mirrored grid
  // rows i and G - i, so the recurrence region is contracted for the rows
  // i < nrows_fold only, split into even and odd degrees (half the work)
  bool fold = false;
  int64_t nrows_fold = 0;
  // alpha = beta = 1/2 exact expansion (cjt_plan_desc.half_k): forward = the
  // U -> T conversion kernel; inverse = synthesis + one chirp-z written
  // straight to the output (no recurrence rows)
  bool half_exact = false;
  double* half_k = nullptr;
  // inverse, moderate N: exact conversion + bf16 tensor-core correction with
  // the per-plan matrix M, row-major [m][k] (cjt_half.cu, cjt_umma.cu), built
  // from edge + blocks[0]
  bool half_gemm = false;
  void* gemm_X = nullptr;
  // grid angles and (alpha, beta) on the device: modulation diagonals built here
  PlanGrid grid{};
  int64_t rec_rows() const { return fold ? nrows_fold : nrows; }
  InvItem* iitems = nullptr;
  int64_t n_iitems = 0;
  int32_t* tile_ids = nullptr;
  void* inv_gen = nullptr;      // K2 generator stream (GenState per row tile x thread)
  int32_t* d_gn0 = nullptr;     // n0 of each work-list row tile (inverse)
  // two-pass contraction: P blocks generated per execution in chunks that fit
  // the per-stream workspace arena, each chunk followed by its DMMA GEMM
  struct Chunk {
    int64_t b0, b1;             // forward: blk_tj range; inverse: work-list row tiles g
    GemmItem* items;
    int64_t n_items;
  };
  bool two_pass = false;
  std::vector<Chunk> chunks;
  int2* blk_tj = nullptr;       // forward P blocks (tile, stage)
  int64_t chunk_bytes = 0;      // largest chunk's P bytes
  int32_t* dt_slot0 = nullptr;
  int32_t* dt_nslot = nullptr;
  int64_t n_islots = 0;
  // per-stream mutable workspaces, so concurrent executions of one plan on
  // different streams never share buffers
  struct Workspace {
    std::vector<void*> allocs;
    int64_t batch = 0;
    double* part = nullptr;
    double* vals = nullptr;    // forward values / inverse wv, [B][G+1]
    double* yacc = nullptr;    // inverse block accumulator [B][N+1]
    double* czpart = nullptr;  // chirp-z m-split partials
    double2* scratch = nullptr;
    double2* spec = nullptr;   // tiled chirp-z spectrum sums
    double* io_in = nullptr;
    double* io_out = nullptr;
    void* tbf = nullptr;       // half_gemm: bf16 copy of the input [B][N+1]
    float* corr = nullptr;     // half_gemm: fp32 correction [B][N+1]
    double* htot = nullptr;    // half forward: per-chunk (even, odd) totals
  };
  std::map<cudaStream_t, Workspace> ws;
  std::mutex ws_mu;
  // serialises execute / reserve of one plan across host threads (the
  // enqueue only; kernels of different streams still overlap), so growing
  // the batch-dependent state never races a launch reading it
  std::mutex exec_mu;
  // set once an execution was recorded into a CUDA graph: from then on the
  // batch-dependent buffers are frozen (a growth would free memory the graph
  // still references), and a larger batch is an error
  bool captured = false;
  int64_t workspace_bytes = 0;
  int64_t last_launches = 0;
  int vt = 64;

  ~cjt_plan() {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    for (auto& kv : ws)
      for (void* p : kv.second.allocs) cudaFree(p);
    for (void* p : ws_allocs) cudaFree(p);
    for (void* p : allocs) cudaFree(p);
    cudaSetDevice(cur);
  }
};

// Standalone batched chirp-z product (trig.py's DCT-I / DST-I / Chebyshev
// synthesis and analysis): one ChirpZDev plus its per-stream workspaces.
struct cjt_chirpz_plan {
  std::unique_ptr<cjt_plan> owner;   // allocations, twiddle table
  ChirpZDev cz{};
  int64_t in_len = 0, out_len = 0;
  struct Ws {
    std::vector<void*> allocs;
    int64_t batch = 0;
    double2* scratch = nullptr;
    double* part = nullptr;
    double2* spec = nullptr;
  };
  std::map<cudaStream_t, Ws> ws;
  std::mutex mu;
  ~cjt_chirpz_plan() {
    for (auto& kv : ws)
      for (void* q : kv.second.allocs) cudaFree(q);
  }
};

namespace {

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};

int dalloc(std::vector<void*>& list, void** p, size_t bytes) {
  *p = nullptr;
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(CJT_ENOMEM, std::string("cudaMalloc(") + std::to_string(bytes) +
                                ") failed: " + cudaGetErrorString(e));
  }
  list.push_back(*p);
  return CJT_OK;
}

template <typename T>
int upload(std::vector<void*>& list, T** dst, const T* src, size_t count) {
  void* p = nullptr;
  if (int rc = dalloc(list, &p, count * sizeof(T))) return rc;
  *dst = static_cast<T*>(p);
  // this thread's stream, not the legacy default stream: a legacy-stream copy
  // would wait for the plan kernels other host threads have in flight
  if (count) {
    CJT_CUDA_TRY(cudaMemcpyAsync(p, src, count * sizeof(T), cudaMemcpyHostToDevice, cudaStreamPerThread));
    CJT_CUDA_TRY(cudaStreamSynchronize(cudaStreamPerThread));
  }
  return CJT_OK;
}

// Many host -> device uploads into ONE allocation, synchronised once (plan
// builds: a cudaMalloc and a synchronised copy per table were most of
// configuration 5's plan-build time).  Sources must stay valid until flush();
// add_owned() keeps a temporary alive inside the batch.
struct UploadBatch {
  struct Item {
    void** dst;
    const void* src;
    size_t bytes, off;
  };
  std::vector<Item> items;
  std::vector<std::vector<double>> owned;
  size_t total = 0;
  template <typename T>
  void add(T** dst, const T* src, size_t count) {
    const size_t bytes = count * sizeof(T);
    items.push_back({reinterpret_cast<void**>(dst), src, bytes, total});
    total += (bytes + 255) & ~size_t(255);
  }
  void add_owned(const double** dst, std::vector<double>&& v) {
    owned.push_back(std::move(v));
    add(const_cast<double**>(dst), owned.back().data(), owned.back().size());
  }
  int flush(std::vector<void*>& list) {
    if (items.empty()) return CJT_OK;
    void* base = nullptr;
    if (int rc = dalloc(list, &base, std::max<size_t>(total, 256))) return rc;
    for (const Item& it : items) {
      *it.dst = static_cast<char*>(base) + it.off;
      if (it.bytes)
        CJT_CUDA_TRY(cudaMemcpyAsync(*it.dst, it.src, it.bytes, cudaMemcpyHostToDevice, cudaStreamPerThread));
    }
    CJT_CUDA_TRY(cudaStreamSynchronize(cudaStreamPerThread));
    items.clear();
    owned.clear();
    total = 0;
    return CJT_OK;
  }
};

// Device recurrence tables: the reference's seven (A, B, C, rf+-, 1/rf+-) and
// the FMA-form Reinsch tables A/rf+-, C/rf+- (products with the tabulated
// reciprocals) used by the generation kernels.
void batch_tables(UploadBatch& ub, const double* const src[7], size_t tl, RecTablesDev* tab) {
  *tab = RecTablesDev{};
  tab->n_tab = (int64_t)tl;
  const double** t[7] = {&tab->A, &tab->B, &tab->C, &tab->rfp, &tab->rfm, &tab->rfpi, &tab->rfmi};
  for (int k = 0; k < 7; ++k) ub.add(const_cast<double**>(t[k]), src[k], tl);
  const double* num[4] = {src[0], src[0], src[2], src[2]};
  const double* den[4] = {src[5], src[6], src[5], src[6]};
  const double** dst[4] = {&tab->Ap, &tab->Am, &tab->Cp, &tab->Cm};
  for (int k = 0; k < 4; ++k) {
    std::vector<double> prod(tl);
    for (size_t i = 0; i < tl; ++i) prod[i] = num[k][i] * den[k][i];
    ub.add_owned(dst[k], std::move(prod));
  }
}

int upload_tables(std::vector<void*>& A, const double* const src[7], size_t tl, RecTablesDev* tab) {
  UploadBatch ub;
  batch_tables(ub, src, tl, tab);
  return ub.flush(A);
}

// exp(-2 pi i num / den), long-double accurate
inline void unit_root(int64_t num, int64_t den, double* re, double* im) {
  num %= den;
  if (num < 0) num += den;
  if (2 * num > den) num -= den;
  const long double ang = -2.0L * 3.14159265358979323846264338327950288L * (long double)num / (long double)den;
  *re = (double)cosl(ang);
  *im = (double)sinl(ang);
}

// Twiddle tables shared by every plan of a device (immutable, built once per
// length with long-double trigonometry and kept for the process lifetime):
// L = 8192: exp(-2 pi i u / 8192), u < 8192 (+ packed power tables); multi-pass L: the hi table
// exp(-2 pi i a 4096 / L), a < max(1, L / 4096), followed by the lo table
// exp(-2 pi i b / L), b < 4096.
// col_log1 > 0 (multi-pass L with register column passes): followed by the
// column twiddles [p][n2] = exp(-2 pi i n2 2^p / L), p < col_log1, n2 < L >> col_log1
// (coalesced per-lane loads in k_chirpz_cols_fwd_reg)
int shared_twiddles(int64_t L, const double2** out, int col_log1 = 0) {
  static std::map<std::pair<int, int64_t>, void*> cache;
  static std::mutex mu;
  int dev = 0;
  CJT_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({dev, L * 64 + col_log1});
  if (it == cache.end()) {
    std::vector<double2> tw;
    if (L == 8192) {
      // followed by the packed power tables exp(-2 pi i k / 2^c) at
      // 8192 + 2^c + k (tw_pow, cjt_internal.cuh): decimations of the same values
      tw.resize(TW_TABLE_ENTRIES);
      for (int u = 0; u < 8192; ++u) unit_root(u, 8192, &tw[u].x, &tw[u].y);
      for (int c = 0; c <= 13; ++c)
        for (int k = 0; k < (1 << c); ++k) tw[TW_PACKED_OFFSET + (1 << c) + k] = tw[(size_t)k << (13 - c)];
    } else {
      const int64_t nhi = std::max<int64_t>(1, L / 4096);
      tw.resize((size_t)(nhi + 4096));
      for (int64_t a = 0; a < nhi; ++a) unit_root(a * 4096, L, &tw[a].x, &tw[a].y);
      for (int64_t b = 0; b < 4096; ++b) unit_root(b, L, &tw[nhi + b].x, &tw[nhi + b].y);
      if (col_log1 > 0) {
        const int64_t L2 = L >> col_log1;
        tw.resize((size_t)(nhi + 4096 + col_log1 * L2));
        for (int p = 0; p < col_log1; ++p)
          for (int64_t n2 = 0; n2 < L2; ++n2) {
            double2& w = tw[(size_t)(nhi + 4096 + p * L2 + n2)];
            unit_root((n2 << p) % L, L, &w.x, &w.y);
          }
      }
    }
    void* p = nullptr;
    CJT_CUDA_TRY(cudaMalloc(&p, tw.size() * sizeof(double2)));
    CJT_CUDA_TRY(cudaMemcpy(p, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
    it = cache.emplace(std::make_pair(dev, L * 64 + col_log1), p).first;
  }
  *out = (const double2*)it->second;
  return CJT_OK;
}

int log2_exact(int64_t v) {
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return ((int64_t(1) << l) == v) ? l : -1;
}

int build_chirpz(cjt_plan* P, const cjt_chirpz_desc& d, ChirpZDev* out) {
  ChirpZDev cz{};
  cz.p0 = d.p0;
  cz.width = d.width;
  cz.q0 = d.q0;
  cz.qout = d.q0 - d.out_shift;
  cz.count = d.count;
  cz.length = d.length;
  cz.m_count = d.m_count;
  cz.accumulate = d.accumulate;
  const int lg = log2_exact(d.length);
  if (lg < 4 || lg > 26) return fail(CJT_EINVAL, "chirp-z length must be a power of two in [16, 2^26]");
  if (d.width < 1 || d.count < 1 || d.m_count < 1 || d.n_tiles_in < 1 || d.n_tiles_out < 1)
    return fail(CJT_EINVAL, "inconsistent chirp-z descriptor");
  if (cz.qout < 0) return fail(CJT_EINVAL, "chirp-z out_shift exceeds q0");
  const bool tiled = d.n_tiles_in > 1 || d.n_tiles_out > 1;
  if (tiled && lg > 13 && d.n_tiles_in > 1 && d.n_tiles_out > 1)
    return fail(CJT_EINVAL, "tiled multi-pass chirp-z needs n_tiles_in == 1 or n_tiles_out == 1");
  {
    int64_t wsum = 0, csum = 0, wmax = 0, cmax = 0;
    for (int i = 0; i < d.n_tiles_in; ++i) {
      if (d.tiles_in[2 * i] != wsum) return fail(CJT_EINVAL, "input tiles must be contiguous");
      wsum += d.tiles_in[2 * i + 1];
      wmax = std::max(wmax, d.tiles_in[2 * i + 1]);
    }
    for (int j = 0; j < d.n_tiles_out; ++j) {
      if (d.tiles_out[2 * j] != csum) return fail(CJT_EINVAL, "output tiles must be contiguous");
      csum += d.tiles_out[2 * j + 1];
      cmax = std::max(cmax, d.tiles_out[2 * j + 1]);
    }
    if (wsum != d.width || csum != d.count || wmax + cmax - 1 > d.length)
      return fail(CJT_EINVAL, "chirp-z tiles do not cover the index rectangle");
  }
  cz.n_in = d.n_tiles_in;
  cz.n_out = d.n_tiles_out;
  cz.count_max = 0;
  for (int j = 0; j < d.n_tiles_out; ++j) cz.count_max = std::max<int64_t>(cz.count_max, d.tiles_out[2 * j + 1]);
  if (int rc = upload(P->allocs, const_cast<int64_t**>(&cz.tin), d.tiles_in, (size_t)2 * d.n_tiles_in)) return rc;
  if (int rc = upload(P->allocs, const_cast<int64_t**>(&cz.tout), d.tiles_out, (size_t)2 * d.n_tiles_out)) return rc;
  cz.log2len = lg;
  const size_t nm = (size_t)d.m_count;
  const bool cluster = lg >= 14 && lg <= 17 && !tiled && cluster_enabled();
  if (lg >= 14 && !cluster) {
    // on-chip rows (two-level FFT) and short columns: wide,
    // coalesced column tiles (E / L1 columns) in passes 1 and 3
    // rows: 8192 points (1 CTA/SM) only for 2^14 / 2^15 (columns of 2 / 4
    // points would be too short otherwise); from 2^16 on, 4096-point rows at
    // 2 CTAs/SM overlap their HBM and FFT phases and win despite longer
    // columns.  $CJT_MP_L2MAX (experiments) caps the row length.
    static const int l2max = [] {
      const char* e = getenv("CJT_MP_L2MAX");
      return e ? std::max(10, std::min(13, atoi(e))) : 13;
    }();
    // (8192-point rows only while the columns would otherwise fall below 16
    // points: 4096-point rows at 2 CTAs/SM win for 2^16 .. 2^19 too, config-4/5
    // A/B with CJT_MP_L2MAX: 58.9 -> 57.8 ms, 159.4 -> 155.5 ms)
    int l2 = std::min({l2max, lg - 4, lg >= 16 ? 12 : 13});
    {   // $CJT_MP_L2_<lg>=<l2> (experiments): row length of one Bluestein length
      const std::string key = "CJT_MP_L2_" + std::to_string(lg);
      if (const char* e = getenv(key.c_str())) l2 = std::max(10, std::min({13, lg - 4, atoi(e)}));
    }
    cz.log1 = lg - l2;
    cz.log2 = l2;
  }
  // spectrum layout of the executing kernels: natural (cluster, short fused
  // tiles), two-level on-chip order (fused tiles >= 512), multi-pass rows
  // [k1][k2] with the rows' own order
  const int mode = cluster ? 0 : lg <= 13 ? (fft2_used(lg) ? 1 : 0) : (fft2_used(cz.log2) ? 3 : 2);
  const int ntile = d.n_tiles_in * d.n_tiles_out;
  if (d.device_tables) {
    // device-side planning: chirps, folded diagonals, spectra (cjt_plan_dev.cu)
    const int64_t G = d.grid_g;
    if (G < 1) return fail(CJT_EINVAL, "device-built chirp-z tables need grid_g >= 1");
    if (int rc = build_device_diag(DevDiag{d.pre_kind, reinterpret_cast<const double2*>(d.pre), d.pre_row0},
                                   d.width, d.m_count, d.p0, G, P->grid, P->allocs, &cz.pre))
      return rc;
    if (int rc = build_device_diag(DevDiag{d.post_kind, reinterpret_cast<const double2*>(d.post), d.post_row0},
                                   d.count, d.m_count, d.q0, G, P->grid, P->allocs, &cz.post))
      return rc;
    if (int rc = build_device_spectra(cz, cz.tin, cz.tout, G, mode, P->allocs, &cz.khat)) return rc;
  } else {
    if (int rc = upload(P->allocs, const_cast<double2**>(&cz.pre),
                        reinterpret_cast<const double2*>(d.pre), nm * d.width)) return rc;
    if (int rc = upload(P->allocs, const_cast<double2**>(&cz.post),
                        reinterpret_cast<const double2*>(d.post), nm * d.count)) return rc;
    if (int rc = permute_spectra(reinterpret_cast<const double2*>(d.kernel_hat), d.length, ntile, mode, cz.log1,
                                 cz.log2, P->allocs, &cz.khat))
      return rc;
  }
  if (lg >= 14) {
    const double2* t = nullptr;
    const int col_log1 = (!cluster && cz.log1 <= 5) ? cz.log1 : 0;
    if (int rc = shared_twiddles(d.length, &t, col_log1)) return rc;
    cz.tw_hi = t;
    cz.tw_lo = t + std::max<int64_t>(1, d.length / 4096);
    cz.tw_col = col_log1 ? cz.tw_lo + 4096 : nullptr;
  }
  if (lg >= 14 && !cluster) {
    // one slot per input or output tile per (vector, term)
    P->scratch_elems_per_vec = std::max<int64_t>(
        P->scratch_elems_per_vec, d.length * d.m_count * std::max(d.n_tiles_in, d.n_tiles_out));
  }
  // FFTs executed per vector: per term, one forward FFT per input tile and one
  // inverse FFT per output tile; on-chip tiles sum the input tiles' spectra
  // per output tile, multi-pass tiles share the forward FFT across outputs
  const double ffts = lg <= 13 ? (double)d.n_tiles_out * (d.n_tiles_in + 1)
                               : (double)(d.n_tiles_in + d.n_tiles_out);
  P->fft_points += (double)d.m_count * ffts * (double)d.length * lg;
  *out = cz;
  return CJT_OK;
}

bool rec_any(const cjt_plan* P) {
  for (int64_t c : P->h_cut)
    if (c > 0) return true;
  return false;
}

// P chunk size of the two-pass contraction (bytes of generated P per chunk):
// $CJT_PGEN_CHUNK_MB, default 2 GiB; 0 disables the two-pass path.
int64_t pgen_chunk_budget() {
  if (const char* e = getenv("CJT_PGEN_CHUNK_MB")) return (int64_t)atoll(e) << 20;
  return (int64_t)2 << 30;
}

// Per-(device, stream) workspace arena for the P chunks, shared by every plan
// executing on that stream (stream order makes the reuse safe).  Grown outside
// graph capture (first execution on a stream / reserve).
struct Arena {
  void* ptr = nullptr;
  int64_t bytes = 0;
  bool captured = false;   // referenced by a CUDA graph: never freed or grown
};
std::map<std::pair<int, cudaStream_t>, Arena>& arenas() {
  static std::map<std::pair<int, cudaStream_t>, Arena> m;
  return m;
}
std::mutex& arena_mutex() {
  static std::mutex mu;
  return mu;
}
int arena_get(int device, cudaStream_t st, int64_t need, double** out) {
  std::lock_guard<std::mutex> lk(arena_mutex());
  Arena& a = arenas()[{device, st}];
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (a.bytes < need) {
    if (cs != cudaStreamCaptureStatusNone)
      return fail(CJT_EINVAL, "P workspace arena must be grown before graph capture (run once uncaptured)");
    if (a.captured)
      return fail(CJT_EINVAL, "P workspace arena of this stream is referenced by a captured CUDA graph and "
                              "cannot grow; execute the largest plan on this stream before capturing");
    CJT_CUDA_TRY(cudaStreamSynchronize(st));
    if (a.ptr) cudaFree(a.ptr);
    a.ptr = nullptr;
    a.bytes = 0;
    cudaError_t e = cudaMalloc(&a.ptr, (size_t)need);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(CJT_ENOMEM, std::string("arena cudaMalloc failed: ") + cudaGetErrorString(e));
    }
    a.bytes = need;
  }
  if (cs != cudaStreamCaptureStatusNone) a.captured = true;
  *out = (double*)a.ptr;
  return CJT_OK;
}

// Work lists depend on the batch size (split-K is sized to fill the GPU).
std::vector<int64_t> tile_max_cut(const cjt_plan* P, int64_t rows_per_tile) {
  const int64_t nr = P->rec_rows();
  const int64_t ntiles = (nr + rows_per_tile - 1) / rows_per_tile;
  std::vector<int64_t> mx((size_t)ntiles, 0);
  for (int64_t i = 0; i < nr; ++i) {
    const int64_t t = i / rows_per_tile;
    mx[t] = std::max(mx[t], P->h_cut[i]);
  }
  return mx;
}

template <typename T>
int upload_ws(cjt_plan* P, T** dst, const std::vector<T>& v) {
  void* p;
  if (int rc = dalloc(P->ws_allocs, &p, std::max<size_t>(1, v.size()) * sizeof(T))) return rc;
  *dst = (T*)p;
  if (!v.empty()) {
    CJT_CUDA_TRY(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, cudaStreamPerThread));
    CJT_CUDA_TRY(cudaStreamSynchronize(cudaStreamPerThread));
  }
  return CJT_OK;
}

// $CJT_FOLD_TWO_PASS=0 (experiments): folded forward plans stay warp-specialised
bool fold_two_pass_enabled() {
  static const bool on = [] {
    const char* e = getenv("CJT_FOLD_TWO_PASS");
    return !(e && e[0] == '0');
  }();
  return on;
}

int build_items(cjt_plan* P, int64_t batch) {
  const int64_t target = 8 * 148;  // CTAs worth of items to fill 148 SMs several times over
  P->two_pass = false;
  P->vt = pick_vt(batch);
  P->chunks.clear();
  P->chunk_bytes = 0;
  // two-pass (P through HBM, DMMA GEMM without generation on the pipe) only
  // pays at VT = 128; up to 64 vectors per tile the warp-specialised kernels
  // (issue-lean producers) win (config-2 / config-3 launch lists)
  // folded plans: 64-vector tiles at most (two accumulator sets per consumer),
  // no two-pass path
  // (inverse: the mirror rows' wv ring doubles the operand tiles, 16-vector
  // tiles keep two CTAs per SM)
  if (P->fold) P->vt = std::min(P->vt, P->direction == CJT_FORWARD ? 64 : 16);
  // two-pass at 128-vector tiles; folded forward plans at 64-vector tiles
  // (their GEMM holds two accumulator sets) once the batch spans several tiles
  const bool tp = P->fold ? (P->direction == CJT_FORWARD && batch > 64 && fold_two_pass_enabled())
                          : P->vt >= 128;
  const int64_t budget_blocks = tp ? pgen_chunk_budget() / (32 * 128 * 8) : 0;
  const int64_t nbt = (batch + P->vt - 1) / P->vt;
  if (P->direction == CJT_FORWARD) {
    const std::vector<int64_t> tmax = tile_max_cut(P, FWD_ROWS);
    const int64_t ntiles = (int64_t)tmax.size();
    double total = 0.0;
    for (int64_t t = 0; t < ntiles; ++t) total += (double)tmax[t];
    int64_t seg = (int64_t)std::ceil(total * nbt / target);
    seg = std::max<int64_t>(8 * FWD_KS, ((seg + FWD_KS - 1) / FWD_KS) * FWD_KS);
    std::vector<FwdItem> items;
    std::vector<int32_t> s0((size_t)ntiles), ns((size_t)ntiles);
    int32_t slot = 0;
    for (int64_t t = 0; t < ntiles; ++t) {
      s0[t] = slot;
      const int64_t top = ((tmax[t] + FWD_KS - 1) / FWD_KS) * FWD_KS;
      int32_t cnt = 0;
      for (int64_t nb = 0; nb < top; nb += seg) {
        FwdItem it{};
        it.row0 = (int32_t)(t * FWD_ROWS);
        it.nrows = (int32_t)std::min<int64_t>(FWD_ROWS, P->rec_rows() - t * FWD_ROWS);
        it.n_begin = (int32_t)nb;
        it.n_end = (int32_t)std::min(top, nb + seg);
        it.slot = slot++;
        items.push_back(it);
        ++cnt;
      }
      ns[t] = cnt;
    }
    // heaviest items first so the tail of the grid is short
    std::stable_sort(items.begin(), items.end(), [](const FwdItem& a, const FwdItem& b) {
      return (a.n_end - a.n_begin) > (b.n_end - b.n_begin);
    });
    // two-pass layout: P blocks (tile t, stage j) for j < ceil(maxcut_t / 32),
    // cut into chunks of whole tiles of at most budget_blocks blocks
    if (budget_blocks > 0) {
      std::vector<int64_t> base((size_t)ntiles + 1, 0);
      std::vector<int2> tj;
      for (int64_t t = 0; t < ntiles; ++t) {
        const int64_t nst = (tmax[t] + FWD_KS - 1) / FWD_KS;
        base[t + 1] = base[t] + nst;
        for (int64_t j = 0; j < nst; ++j) tj.push_back(make_int2((int)t, (int)j));
      }
      bool ok = true;
      std::vector<std::pair<int64_t, int64_t>> tranges;   // [t0, t1) per chunk
      for (int64_t t0 = 0; t0 < ntiles && ok;) {
        int64_t t1 = t0;
        while (t1 < ntiles && (base[t1 + 1] - base[t0]) <= budget_blocks) ++t1;
        if (t1 == t0) ok = false;   // a single tile exceeds the budget
        tranges.push_back({t0, t1});
        t0 = t1;
      }
      if (ok && !tj.empty()) {
        if (int rc = upload_ws(P, &P->blk_tj, tj)) return rc;
        for (auto [t0, t1] : tranges) {
          std::vector<GemmItem> gi;
          for (const FwdItem& it : items) {
            const int64_t t = it.row0 / FWD_ROWS;
            if (t < t0 || t >= t1) continue;
            GemmItem g{};
            g.p_block0 = base[t] - base[t0] + it.n_begin / FWD_KS;
            g.x_off0 = it.n_begin;
            g.ids_off = -1;
            g.nstages = (it.n_end - it.n_begin) / FWD_KS;
            g.slot = it.slot;
            gi.push_back(g);
          }
          cjt_plan::Chunk ch{base[t0], base[t1], nullptr, (int64_t)gi.size()};
          if (int rc = upload_ws(P, &ch.items, gi)) return rc;
          P->chunks.push_back(ch);
          P->chunk_bytes = std::max<int64_t>(P->chunk_bytes, (base[t1] - base[t0]) * 32 * 128 * 8);
        }
        P->two_pass = true;
      }
    }
    if (int rc = upload_ws(P, &P->fitems, items)) return rc;
    if (int rc = upload_ws(P, &P->tile_slot0, s0)) return rc;
    if (int rc = upload_ws(P, &P->tile_nslot, ns)) return rc;
    P->n_fitems = (int64_t)items.size();
    P->n_fslots = slot;
  } else {
    const std::vector<int64_t> tmax = tile_max_cut(P, INV_RT);
    const int64_t ntiles = (int64_t)tmax.size();
    const int64_t ndeg = P->n + 1;
    const int64_t nd = (ndeg + INV_DT - 1) / INV_DT;
    std::vector<std::vector<int32_t>> active((size_t)nd);
    int64_t total_active = 0;
    for (int64_t d = 0; d < nd; ++d) {
      for (int64_t t = 0; t < ntiles; ++t)
        if (tmax[t] > d * INV_DT) active[d].push_back((int32_t)t);
      total_active += (int64_t)active[d].size();
    }
    const int64_t cs = std::max<int64_t>(1, (int64_t)std::ceil((double)total_active * nbt / target));
    std::vector<InvItem> items;
    std::vector<int32_t> ids, gn0, s0((size_t)nd), ns((size_t)nd);
    int32_t slot = 0;
    for (int64_t d = 0; d < nd; ++d) {
      s0[d] = slot;
      const int64_t na = (int64_t)active[d].size();
      // split the active row tiles of this degree tile into near-equal chunks of <= cs
      const int64_t nchunks = std::max<int64_t>(1, (na + cs - 1) / cs);
      int32_t cnt = 0;
      for (int64_t q = 0; q < nchunks && na > 0; ++q) {
        const int64_t a0 = na * q / nchunks, a1 = na * (q + 1) / nchunks;
        if (a1 <= a0) continue;
        InvItem it{};
        it.n0 = (int32_t)(d * INV_DT);
        it.t_begin = (int32_t)ids.size();
        for (int64_t a = a0; a < a1; ++a) {
          ids.push_back(active[d][a]);
          gn0.push_back((int32_t)(d * INV_DT));
        }
        it.t_count = (int32_t)(a1 - a0);
        it.slot = slot++;
        items.push_back(it);
        ++cnt;
      }
      ns[d] = cnt;
    }
    std::stable_sort(items.begin(), items.end(),
                     [](const InvItem& a, const InvItem& b) { return a.t_count > b.t_count; });
    if (budget_blocks > 0 && !items.empty()) {
      // chunks of whole items over the work-list row tiles g (items own
      // disjoint contiguous g ranges), each at most budget_blocks tiles
      std::vector<InvItem> by_g = items;
      std::stable_sort(by_g.begin(), by_g.end(),
                       [](const InvItem& a, const InvItem& b) { return a.t_begin < b.t_begin; });
      bool ok = true;
      size_t i0 = 0;
      std::vector<cjt_plan::Chunk> chs;
      std::vector<std::vector<GemmItem>> chitems;
      while (i0 < by_g.size() && ok) {
        const int64_t g0 = by_g[i0].t_begin;
        size_t i1 = i0;
        while (i1 < by_g.size() && (by_g[i1].t_begin + by_g[i1].t_count - g0) <= budget_blocks) ++i1;
        if (i1 == i0) {
          ok = false;
          break;
        }
        const int64_t g1 = by_g[i1 - 1].t_begin + by_g[i1 - 1].t_count;
        std::vector<GemmItem> gi;
        for (size_t q = i0; q < i1; ++q) {
          GemmItem g{};
          g.p_block0 = by_g[q].t_begin - g0;
          g.x_off0 = 0;
          g.ids_off = by_g[q].t_begin;
          g.nstages = by_g[q].t_count;
          g.slot = by_g[q].slot;
          gi.push_back(g);
        }
        std::stable_sort(gi.begin(), gi.end(),
                         [](const GemmItem& a, const GemmItem& b) { return a.nstages > b.nstages; });
        chs.push_back(cjt_plan::Chunk{g0, g1, nullptr, (int64_t)gi.size()});
        chitems.push_back(std::move(gi));
        i0 = i1;
      }
      if (ok) {
        for (size_t c = 0; c < chs.size(); ++c) {
          if (int rc = upload_ws(P, &chs[c].items, chitems[c])) return rc;
          P->chunk_bytes = std::max<int64_t>(P->chunk_bytes, (chs[c].b1 - chs[c].b0) * INV_RT * INV_DT * 8);
        }
        P->chunks = chs;
        P->two_pass = true;
      }
    }
    if (int rc = upload_ws(P, &P->iitems, items)) return rc;
    if (int rc = upload_ws(P, &P->tile_ids, ids)) return rc;
    int32_t* d_gn0 = nullptr;
    if (int rc = upload_ws(P, &d_gn0, gn0)) return rc;
    P->d_gn0 = d_gn0;
    void* gp = nullptr;
    const int64_t total = (int64_t)ids.size();
    if (int rc = dalloc(P->ws_allocs, &gp, (size_t)std::max<int64_t>(total, 1) * 128 * GEN_STATE_BYTES)) return rc;
    P->inv_gen = gp;
    if (int rc = launch_build_inv_gen(P->rows, P->ck_off, P->ck, P->tile_ids, d_gn0, total, gp, 0)) return rc;
    CJT_CUDA_TRY(cudaDeviceSynchronize());
    if (int rc = upload_ws(P, &P->dt_slot0, s0)) return rc;
    if (int rc = upload_ws(P, &P->dt_nslot, ns)) return rc;
    P->n_iitems = (int64_t)items.size();
    P->n_islots = slot;
  }
  return CJT_OK;
}

void free_workspace(cjt_plan* P) {
  for (void* p : P->ws_allocs) cudaFree(p);
  P->ws_allocs.clear();
  P->reserved = 0;
  P->workspace_bytes = 0;
}

// caller holds P->exec_mu
int reserve(cjt_plan* P, int64_t batch) {
  if (batch <= P->reserved) return CJT_OK;
  if (P->captured)
    return fail(CJT_EINVAL, "plan is referenced by a captured CUDA graph (reserved batch " +
                                std::to_string(P->reserved) + "); growing it to " + std::to_string(batch) +
                                " would free buffers the graph uses: reserve the largest batch before capture");
  CJT_CUDA_TRY(cudaDeviceSynchronize());
  free_workspace(P);
  {
    std::lock_guard<std::mutex> lk(P->ws_mu);
    for (auto& kv : P->ws)
      for (void* q : kv.second.allocs) cudaFree(q);
    P->ws.clear();
  }
  if (int rc = build_items(P, batch)) return rc;
  P->reserved = batch;
  return CJT_OK;
}

// workspace of `st`, allocated on first use (outside graph capture)
int get_workspace(cjt_plan* P, cudaStream_t st, cjt_plan::Workspace** out) {
  std::lock_guard<std::mutex> lk(P->ws_mu);
  cjt_plan::Workspace& W = P->ws[st];
  *out = &W;
  if (W.batch >= P->reserved) return CJT_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs != cudaStreamCaptureStatusNone)
    return fail(CJT_EINVAL, "plan workspace for this stream must exist before graph capture (run once uncaptured)");
  for (void* q : W.allocs) cudaFree(q);
  W = cjt_plan::Workspace{};
  const int64_t batch = P->reserved;
  const int64_t G1 = P->G + 1, N1 = P->n + 1;
  void* p;
  int64_t bytes = 0;
  if (P->half_gemm) {
    if (int rc = half_gemm_prepare(st)) return rc;
    if (int rc = dalloc(W.allocs, &p, (size_t)(N1 * batch) * 2)) return rc;
    W.tbf = p;
    if (int rc = dalloc(W.allocs, &p, (size_t)(N1 * batch) * 4)) return rc;
    W.corr = (float*)p;
    if (int rc = dalloc(W.allocs, &p, (size_t)(N1 * batch) * 8)) return rc;
    W.io_in = (double*)p;
    if (int rc = dalloc(W.allocs, &p, (size_t)(N1 * batch) * 8)) return rc;
    W.io_out = (double*)p;
    W.batch = batch;
    P->workspace_bytes = std::max<int64_t>(P->workspace_bytes, N1 * batch * 22);
    return CJT_OK;
  }
  const int64_t part_elems = (P->direction == CJT_FORWARD) ? P->n_fslots * FWD_ROWS * (P->fold ? 2 : 1)
                                                            : P->n_islots * INV_DT;
  if (int rc = dalloc(W.allocs, &p, (size_t)(part_elems * batch) * 8)) return rc;
  W.part = (double*)p;
  bytes += part_elems * batch * 8;
  if (P->half_exact && P->direction == CJT_FORWARD && half_forward_scratch(N1) > 0) {
    if (int rc = dalloc(W.allocs, &p, (size_t)(half_forward_scratch(N1) * batch) * 8)) return rc;
    W.htot = (double*)p;
    bytes += half_forward_scratch(N1) * batch * 8;
  }
  if (!(P->half_exact && P->direction == CJT_FORWARD)) {   // the exact forward needs no grid values
    if (int rc = dalloc(W.allocs, &p, (size_t)(G1 * batch) * 8)) return rc;
    W.vals = (double*)p;
    bytes += G1 * batch * 8;
  }
  if (P->direction == CJT_INVERSE && !P->blocks.empty() && !P->half_exact) {
    if (int rc = dalloc(W.allocs, &p, (size_t)(N1 * batch) * 8)) return rc;
    W.yacc = (double*)p;
    bytes += N1 * batch * 8;
  }
  if (P->scratch_elems_per_vec > 0) {
    if (int rc = dalloc(W.allocs, &p, (size_t)(P->scratch_elems_per_vec * batch) * 16)) return rc;
    W.scratch = (double2*)p;
    bytes += P->scratch_elems_per_vec * batch * 16;
  }
  int64_t cz_part = 0, cz_spec = 0;
  {
    std::vector<const ChirpZDev*> czs;
    if (P->edge.length > 0) czs.push_back(&P->edge);
    for (const ChirpZDev& cz : P->blocks) czs.push_back(&cz);
    for (const ChirpZDev* cz : czs) {
      int64_t pe, se;
      chirpz_workspace(*cz, batch, &pe, &se);
      cz_part = std::max(cz_part, pe);
      cz_spec = std::max(cz_spec, se);
    }
  }
  if (cz_part > 0) {
    if (int rc = dalloc(W.allocs, &p, (size_t)cz_part * 8)) return rc;
    W.czpart = (double*)p;
    bytes += cz_part * 8;
  }
  if (cz_spec > 0) {
    if (int rc = dalloc(W.allocs, &p, (size_t)cz_spec * 16)) return rc;
    W.spec = (double2*)p;
    bytes += cz_spec * 16;
  }
  if (int rc = dalloc(W.allocs, &p, (size_t)(N1 * batch) * 8)) return rc;
  W.io_in = (double*)p;
  if (int rc = dalloc(W.allocs, &p, (size_t)(N1 * batch) * 8)) return rc;
  W.io_out = (double*)p;
  bytes += 2 * N1 * batch * 8;
  W.batch = batch;
  P->workspace_bytes = std::max<int64_t>(P->workspace_bytes, bytes);
  return CJT_OK;
}

// stage mask: CJT_STAGE_REC (recurrence contraction + its reduction),
// CJT_STAGE_BLOCKS (asymptotic-block chirp-z), CJT_STAGE_EDGE (analysis /
// synthesis chirp-z).  Partial masks are for timing individual kernels only.
int execute(cjt_plan* P, const double* in, double* out, int64_t batch, cudaStream_t st,
            int stages = CJT_STAGE_ALL) {
  {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs != cudaStreamCaptureStatusNone) P->captured = true;
  }
  cjt_plan::Workspace* Wp = nullptr;
  if (int rc = get_workspace(P, st, &Wp)) return rc;
  cjt_plan::Workspace& W = *Wp;
  int launches = 0;
  const int64_t N1 = P->n + 1, G1 = P->G + 1;
  const bool rec = stages & CJT_STAGE_REC, blk = stages & CJT_STAGE_BLOCKS, edge = stages & CJT_STAGE_EDGE;
  if (P->half_exact && P->direction == CJT_FORWARD) {
    if (rec) {
      if (int rc = launch_half_forward(in, N1, out, N1, P->half_k, N1, batch, W.htot, st)) return rc;
      launches += half_forward_scratch(N1) > 0 ? 2 : 1;
    }
  } else if (P->half_gemm) {
    if (blk) {
      if (int rc = half_gemm_inverse(in, out, N1, batch, P->gemm_X, W.tbf, W.corr, P->half_k, st)) return rc;
      launches += 3;
    }
  } else if (P->half_exact) {
    if (edge)
      if (int rc = launch_chirpz(P->edge, P->tw8192, in, N1, W.vals, G1, batch, W.scratch, W.czpart, W.spec, st, &launches))
        return rc;
    if (blk)
      for (const ChirpZDev& cz : P->blocks)
        if (int rc = launch_chirpz(cz, P->tw8192, W.vals, G1, out, N1, batch, W.scratch, W.czpart, W.spec, st, &launches))
          return rc;
  } else if (P->direction == CJT_FORWARD) {
    if (rec && P->two_pass) {
      double* pw = nullptr;
      if (int rc = arena_get(P->device, st, P->chunk_bytes, &pw)) return rc;
      for (const auto& ch : P->chunks) {
        if (int rc = launch_pgen_fwd(P->rows, P->tab, P->ck_off, P->ck, P->blk_tj + ch.b0, ch.b1 - ch.b0, pw,
                                     P->fold, st))
          return rc;
        if (int rc = launch_rec_gemm(ch.items, ch.n_items, pw, nullptr, in, N1, N1, batch, P->vt, false,
                                     P->fold, W.part, st)) return rc;
        launches += 2;
      }
      launches -= 1;
    } else if (rec) {
      if (int rc = launch_rec_forward(P->rows, P->tab, P->ck_off, P->ck, P->fitems, P->n_fitems, in, N1,
                                      N1, batch, P->vt, P->fold, W.part, st)) return rc;
    }
    if (rec) {
      if (int rc = launch_rec_forward_reduce(P->tile_slot0, P->tile_nslot, P->rec_rows(), W.part, W.vals,
                                             G1, batch, P->G, P->fold, st)) return rc;
      launches += 2;
    }
    if (blk)
      for (const ChirpZDev& cz : P->blocks)
        if (int rc = launch_chirpz(cz, P->tw8192, in, N1, W.vals, G1, batch, W.scratch, W.czpart, W.spec, st, &launches))
          return rc;
    if (edge)
      if (int rc = launch_chirpz(P->edge, P->tw8192, W.vals, G1, out, N1, batch, W.scratch, W.czpart, W.spec, st, &launches))
        return rc;
  } else {
    if (edge)
      if (int rc = launch_chirpz(P->edge, P->tw8192, in, N1, W.vals, G1, batch, W.scratch, W.czpart, W.spec, st, &launches))
        return rc;
    if (blk && !P->blocks.empty()) {
      CJT_CUDA_TRY(cudaMemsetAsync(W.yacc, 0, (size_t)(N1 * batch) * 8, st));
      for (const ChirpZDev& cz : P->blocks)
        if (int rc = launch_chirpz(cz, P->tw8192, W.vals, G1, W.yacc, N1, batch, W.scratch, W.czpart, W.spec, st, &launches))
          return rc;
    }
    if (rec && P->two_pass) {
      double* pw = nullptr;
      if (int rc = arena_get(P->device, st, P->chunk_bytes, &pw)) return rc;
      for (const auto& ch : P->chunks) {
        if (int rc = launch_pgen_inv(P->tab, P->inv_gen, P->d_gn0, ch.b0, ch.b1, pw, st)) return rc;
        if (int rc = launch_rec_gemm(ch.items, ch.n_items, pw, P->tile_ids, W.vals, G1, G1, batch, P->vt, true,
                                     false, W.part, st)) return rc;
        launches += 2;
      }
      launches -= 1;
    } else if (rec) {
      if (int rc = launch_rec_inverse(P->tab, P->inv_gen, P->rec_rows(), P->iitems, P->n_iitems, P->tile_ids,
                                      W.vals, G1, batch, P->vt, P->fold, P->G, W.part, st)) return rc;
    }
    if (rec) {
      if (int rc = launch_inverse_finish(P->dt_slot0, P->dt_nslot, N1, W.part, W.yacc, P->scal, out, N1,
                                         batch, st)) return rc;
      launches += 2;
    }
  }
  if (stages == CJT_STAGE_ALL) P->last_launches = launches;
  return CJT_OK;
}

// M of a half_gemm plan: M e_b for the unit vectors e_b, in chunks, through
// the plan's synthesis (edge) and correction (blocks[0]) chirp-z products,
// rounded to bf16 (row b of X = column b of M), then transposed in place to
// row-major M[m][k] (gemm_X).
int build_half_gemm_matrix(cjt_plan* P) {
  const int64_t n1 = P->n + 1, G1 = P->G + 1;
  CJT_CUDA_TRY(cudaStreamSynchronize(cudaStreamPerThread));   // tables built on this thread's stream
  const int64_t chunk = std::min<int64_t>(n1, 512);
  std::vector<void*> tmp;
  struct Free {
    std::vector<void*>* v;
    ~Free() { for (void* q : *v) cudaFree(q); }
  } fr{&tmp};
  void* p;
  if (int rc = dalloc(P->allocs, &p, (size_t)(n1 * n1) * 2)) return rc;
  P->gemm_X = p;
  double *ein, *eout, *vals, *part = nullptr;
  double2 *scratch = nullptr, *spec = nullptr;
  if (int rc = dalloc(tmp, &p, (size_t)(chunk * n1) * 8)) return rc;
  ein = (double*)p;
  if (int rc = dalloc(tmp, &p, (size_t)(chunk * n1) * 8)) return rc;
  eout = (double*)p;
  if (int rc = dalloc(tmp, &p, (size_t)(chunk * G1) * 8)) return rc;
  vals = (double*)p;
  if (P->scratch_elems_per_vec > 0) {
    if (int rc = dalloc(tmp, &p, (size_t)(P->scratch_elems_per_vec * chunk) * 16)) return rc;
    scratch = (double2*)p;
  }
  int64_t pe = 0, se = 0;
  for (const ChirpZDev* cz : {&P->edge, &P->blocks[0]}) {
    int64_t a, b;
    chirpz_workspace(*cz, chunk, &a, &b);
    pe = std::max(pe, a);
    se = std::max(se, b);
  }
  if (pe > 0) {
    if (int rc = dalloc(tmp, &p, (size_t)pe * 8)) return rc;
    part = (double*)p;
  }
  if (se > 0) {
    if (int rc = dalloc(tmp, &p, (size_t)se * 16)) return rc;
    spec = (double2*)p;
  }
  int launches = 0;
  for (int64_t b0 = 0; b0 < n1; b0 += chunk) {
    const int64_t nb = std::min(chunk, n1 - b0);
    if (int rc = launch_identity(ein, n1, b0, nb, cudaStreamPerThread)) return rc;
    if (int rc = launch_chirpz(P->edge, P->tw8192, ein, n1, vals, G1, nb, scratch, part, spec, cudaStreamPerThread, &launches))
      return rc;
    if (int rc = launch_chirpz(P->blocks[0], P->tw8192, vals, G1, eout, n1, nb, scratch, part, spec, cudaStreamPerThread, &launches))
      return rc;
    if (int rc = launch_to_bf16(eout, n1, (char*)P->gemm_X + (size_t)(b0 * n1) * 2, n1, n1, nb, cudaStreamPerThread)) return rc;
  }
  // row-major M[m][k] (K-major operand of the tensor-core GEMM): transpose X
  if (int rc = dalloc(tmp, &p, (size_t)(n1 * n1) * 2)) return rc;
  if (int rc = launch_transpose_bf16(P->gemm_X, p, n1, n1, cudaStreamPerThread)) return rc;
  CJT_CUDA_TRY(cudaMemcpyAsync(P->gemm_X, p, (size_t)(n1 * n1) * 2, cudaMemcpyDeviceToDevice, cudaStreamPerThread));
  CJT_CUDA_TRY(cudaStreamSynchronize(cudaStreamPerThread));   // before the temporaries are freed
  return CJT_OK;
}

// DFMA throughput probe: independent FMA chains, no memory traffic.
__global__ void k_fp64_probe(double* sink, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
  double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
  const double m = 0.999999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 1234.5) sink[threadIdx.x] = s;
}

}  // namespace

extern "C" {

int cjt_version(void) { return 1; }

const char* cjt_last_error(void) { return cjt::g_last_error.c_str(); }

int cjt_device_count(int* count) {
  *count = 0;
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *count = 0;
    return fail(CJT_ENODEV, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  return CJT_OK;
}

int cjt_plan_create(const cjt_plan_desc* d, cjt_plan** out) {
  if (!d || !out) return fail(CJT_EINVAL, "null argument");
  *out = nullptr;
  if (d->direction != CJT_FORWARD && d->direction != CJT_INVERSE) return fail(CJT_EINVAL, "bad direction");
  if (d->n < 1) return fail(CJT_EINVAL, "N must be >= 1");
  const int64_t G = d->grid_n;
  if (G != (d->direction == CJT_FORWARD ? d->n : 2 * d->n)) return fail(CJT_EINVAL, "grid_n inconsistent with direction");
  int ndev = 0;
  if (cjt_device_count(&ndev) || ndev == 0) return fail(CJT_ENODEV, "no CUDA device visible");
  // $CJT_PLAN_TIMING=1 (diagnostics): phase times of this build on stderr
  static const bool timing = [] {
    const char* e = getenv("CJT_PLAN_TIMING");
    return e && e[0] == '1';
  }();
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!timing) return;
    cudaStreamSynchronize(cudaStreamPerThread);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[cjt plan G=%lld] %-12s %8.3f ms\n", (long long)d->grid_n, what,
            std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  std::unique_ptr<cjt_plan> P(new cjt_plan());
  CJT_CUDA_TRY(cudaGetDevice(&P->device));
  P->direction = d->direction;
  P->m_terms = d->m_terms;
  P->n = d->n;
  P->G = G;
  P->nrows = G + 1;
  const int64_t nr = P->nrows;

  P->h_cut.assign(d->cuts, d->cuts + nr);
  int64_t maxcut = 0;
  for (int64_t i = 0; i < nr; ++i) {
    if (P->h_cut[i] < 0) return fail(CJT_EINVAL, "negative cut");
    maxcut = std::max(maxcut, P->h_cut[i]);
    P->rec_steps += P->h_cut[i];
  }
  if (d->table_len < maxcut + 1) return fail(CJT_EINVAL, "recurrence tables shorter than max cut + 1");

  auto& A = P->allocs;
  double *x, *xm;
  int8_t* reg;
  int64_t* cut;
  UploadBatch ub;   // rows, tables and checkpoint offsets: one allocation, one copy
  ub.add(&x, d->x, nr);
  ub.add(&xm, d->xm, nr);
  ub.add(&reg, d->regions, nr);
  ub.add(&cut, d->cuts, nr);
  const size_t tl = (size_t)d->table_len;
  const double* src[7] = {d->A, d->B, d->C, d->rf_plus, d->rf_minus, d->rf_plus_inv, d->rf_minus_inv};
  batch_tables(ub, src, tl, &P->tab);

  // parity folding (alpha = beta): B_n = 0, rf- = -rf+, symmetric cuts,
  // antisymmetric regions.  The forward is insensitive to the mirrored rows'
  // x = -x_i vs the reference's cos(theta_{G-i}) (<= 2e-16 ||c||_1 measured,
  // SURVEY.md 8(c)); the inverse is not (a 1-ulp angle shift moves the
  // alpha = beta = 1/2 inverse by 9e-13 at N = 65535).
  {
    // (the inverse additionally stops at G <= 65534, see below)
    bool sym = d->direction == CJT_FORWARD || G <= 65534;
    for (size_t n = 0; sym && n < tl; ++n)
      sym = d->B[n] == 0.0 && d->rf_minus[n] == -d->rf_plus[n];
    for (int64_t i = 0; sym && i < nr; ++i)
      sym = P->h_cut[i] == P->h_cut[G - i] && d->regions[i] == -d->regions[G - i];
    // the inverse folds only on request ($CJT_FOLD_INVERSE=1): the exact
    // mirror x_{G-i} = -x_i differs from the reference's cos(theta_{G-i}) by
    // ~1e-13 relative near x = -1, which moves the (sensitive) inverse by up
    // to ~2e-13 ||c||_1 (config 5, N <= 2047) -- inside the 1e-12 tolerance
    // but too close to it at large N; the forward moves by <= 2e-16.
    const char* e = getenv("CJT_FOLD");
    const char* ei = getenv("CJT_FOLD_INVERSE");
    P->fold = sym && !(e && e[0] == '0') &&
              (d->direction == CJT_FORWARD || (ei && ei[0] == '1'));
    P->nrows_fold = G / 2 + 1;   // rows 0 .. G/2 (G even: the middle row is its own mirror)
  }

  phase("upload");
  // recurrence checkpoints every CK degrees
  std::vector<int64_t> off((size_t)nr);
  int64_t tot = 0;
  for (int64_t i = 0; i < nr; ++i) {
    off[i] = tot;
    const int64_t c = P->h_cut[i];
    tot += (c >= 1) ? (c - 1) / CK : 0;
  }
  P->ck_count = tot;
  ub.add(&P->ck_off, off.data(), off.size());
  if (int rc = ub.flush(A)) return rc;
  P->rows = RecRowsDev{x, xm, reg, cut, nr};
  void* p;
  if (int rc = dalloc(A, &p, (size_t)std::max<int64_t>(tot, 1) * sizeof(double2))) return rc;
  P->ck = (double2*)p;
  if (tot > 0) {
    if (int rc = launch_checkpoints(P->rows, P->tab, P->ck_off, P->ck, cudaStreamPerThread)) return rc;
  }

  phase("checkpoints");
  // FFT twiddles exp(-2 pi i u / 8192), shared by every plan of the device
  {
    const double2* t = nullptr;
    if (int rc = shared_twiddles(8192, &t)) return rc;
    P->tw8192 = const_cast<double2*>(t);
  }

  if (d->thetas) {
    double* th = nullptr;
    if (int rc = upload(A, &th, d->thetas, (size_t)nr)) return rc;
    // pair weights of the modulation sums (asymptotics.py:22-33)
    std::vector<double> wa((size_t)std::max(1, d->m_terms)), wb(wa.size());
    for (int which = 0; which < 2; ++which) {
      std::vector<double>& w = which ? wb : wa;
      const double gam = which ? d->beta : d->alpha;
      w[0] = 1.0;
      for (size_t l = 1; l < w.size(); ++l) w[l] = w[l - 1] * (0.5 + gam + (double)l - 1) * (0.5 - gam + (double)l - 1) / (double)l;
    }
    double *dwa = nullptr, *dwb = nullptr;
    if (int rc = upload(A, &dwa, wa.data(), wa.size())) return rc;
    if (int rc = upload(A, &dwb, wb.data(), wb.size())) return rc;
    P->grid = PlanGrid{th, dwa, dwb, d->alpha, d->beta};
  }
  if (d->half_k) {
    if (d->direction == CJT_INVERSE && (d->n_blocks != 1 || d->blocks[0].accumulate || rec_any(P.get())))
      return fail(CJT_EINVAL, "exact-expansion inverse plans take one non-accumulating block and no recurrence rows");
    if (d->direction == CJT_FORWARD && (d->n_blocks != 0 || rec_any(P.get())))
      return fail(CJT_EINVAL, "exact-expansion forward plans take no blocks and no recurrence rows");
    P->half_exact = true;
    if (int rc = upload(A, &P->half_k, d->half_k, (size_t)(d->n + 1))) return rc;
  }
  for (int k = 0; k < d->n_blocks; ++k) {
    ChirpZDev cz{};
    if (int rc = build_chirpz(P.get(), d->blocks[k], &cz)) return rc;
    P->blocks.push_back(cz);
  }
  phase("blocks");
  if (d->edge.length > 0) {
    if (int rc = build_chirpz(P.get(), d->edge, &P->edge)) return rc;
    P->has_edge = true;
  } else if (!(P->half_exact && d->direction == CJT_FORWARD)) {
    return fail(CJT_EINVAL, "plan requires an edge (analysis / synthesis) chirp-z");
  }
  if (d->half_gemm) {
    if (!P->half_exact || d->direction != CJT_INVERSE || !P->has_edge)
      return fail(CJT_EINVAL, "half_gemm needs an exact-expansion inverse plan");
    if (int rc = build_half_gemm_matrix(P.get())) return rc;
    P->half_gemm = true;
  }
  if (d->direction == CJT_INVERSE) {
    if (!d->scalings) return fail(CJT_EINVAL, "inverse plan requires scalings");
    if (int rc = upload(A, &P->scal, d->scalings, (size_t)(d->n + 1))) return rc;
  }
  // plan-time kernels ran on this thread's stream (concurrent plan builds on
  // several host threads do not serialise on the legacy stream)
  CJT_CUDA_TRY(cudaStreamSynchronize(cudaStreamPerThread));
  phase("edge+finish");
  *out = P.release();
  return CJT_OK;
}

int cjt_plan_destroy(cjt_plan* plan) {
  if (!plan) return CJT_OK;
  cudaDeviceSynchronize();
  delete plan;
  return CJT_OK;
}

int cjt_plan_reserve(cjt_plan* plan, int64_t max_batch) {
  if (!plan) return fail(CJT_EINVAL, "null plan");
  if (max_batch < 1) return fail(CJT_EINVAL, "batch must be >= 1");
  DeviceGuard g(plan->device);
  std::lock_guard<std::mutex> lk(plan->exec_mu);
  return reserve(plan, max_batch);
}

int cjt_plan_stats_get(const cjt_plan* plan, cjt_plan_stats* s) {
  if (!plan || !s) return fail(CJT_EINVAL, "null argument");
  std::memset(s, 0, sizeof(*s));
  s->launches_per_execute = plan->last_launches;
  s->rec_steps = plan->rec_steps;
  s->checkpoint_bytes = plan->ck_count * 16;
  s->workspace_bytes = plan->workspace_bytes;
  s->reserved_batch = plan->reserved;
  int64_t executed = plan->rec_steps;
  if (plan->fold) {
    executed = 0;
    for (int64_t i = 0; i < plan->nrows_fold; ++i) executed += plan->h_cut[i];
  }
  s->rec_steps_executed = executed;
  s->rec_flops_per_vector = 2.0 * (double)executed;
  s->fft_points_per_vector = plan->fft_points;
  return CJT_OK;
}

// vectors per execution chunk: per-vector grid dimensions (y / z) stay <= 65535
constexpr int64_t kMaxChunk = 65535;

int cjt_execute(cjt_plan* plan, const double* in, double* out, int64_t batch, void* stream) {
  if (!plan || !in || !out) return fail(CJT_EINVAL, "null argument");
  if (batch < 1) return fail(CJT_EINVAL, "batch must be >= 1");
  DeviceGuard g(plan->device);
  std::lock_guard<std::mutex> lk(plan->exec_mu);
  if (int rc = reserve(plan, std::min(batch, kMaxChunk))) return rc;
  const int64_t n1 = plan->n + 1;
  for (int64_t b0 = 0; b0 < batch; b0 += kMaxChunk) {
    const int64_t nb = std::min(kMaxChunk, batch - b0);
    if (int rc = execute(plan, in + b0 * n1, out + b0 * n1, nb, (cudaStream_t)stream)) return rc;
  }
  return CJT_OK;
}

int cjt_execute_stage(cjt_plan* plan, const double* in, double* out, int64_t batch, int32_t stages,
                      void* stream) {
  if (!plan || !in || !out) return fail(CJT_EINVAL, "null argument");
  DeviceGuard g(plan->device);
  std::lock_guard<std::mutex> lk(plan->exec_mu);
  if (batch < 1 || batch > plan->reserved) return fail(CJT_EINVAL, "batch must be in [1, reserved]");
  return execute(plan, in, out, batch, (cudaStream_t)stream, stages);
}

int cjt_probe_fp64_peak(double* tflops, void* stream) {
  if (!tflops) return fail(CJT_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 0;
  CJT_CUDA_TRY(cudaGetDevice(&dev));
  CJT_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* sink = nullptr;
  CJT_CUDA_TRY(cudaMalloc(&sink, 1024 * sizeof(double)));
  const int threads = 512, blocks = sms * 4, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_fp64_probe<<<blocks, threads, 0, st>>>(sink, 64);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0, st);
    k_fp64_probe<<<blocks, threads, 0, st>>>(sink, iters);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  CJT_CUDA_TRY(cudaGetLastError());
  const double flops = 2.0 * 8.0 * 16.0 * iters * (double)threads * blocks;
  *tflops = flops / (best * 1e-3) / 1e12;
  return CJT_OK;
}

int cjt_execute_host(cjt_plan* plan, const double* in_host, double* out_host, int64_t batch,
                     void* stream) {
  if (!plan || !in_host || !out_host) return fail(CJT_EINVAL, "null argument");
  if (batch < 1) return fail(CJT_EINVAL, "batch must be >= 1");
  DeviceGuard g(plan->device);
  std::lock_guard<std::mutex> lk(plan->exec_mu);
  const int64_t chunk = std::min(batch, kMaxChunk);
  if (int rc = reserve(plan, chunk)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  cjt_plan::Workspace* W = nullptr;
  if (int rc = get_workspace(plan, st, &W)) return rc;
  const int64_t n1 = plan->n + 1;
  for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
    const int64_t nb = std::min(chunk, batch - b0);
    const size_t bytes = (size_t)(nb * n1) * 8;
    CJT_CUDA_TRY(cudaMemcpyAsync(W->io_in, in_host + b0 * n1, bytes, cudaMemcpyHostToDevice, st));
    if (int rc = execute(plan, W->io_in, W->io_out, nb, st)) return rc;
    CJT_CUDA_TRY(cudaMemcpyAsync(out_host + b0 * n1, W->io_out, bytes, cudaMemcpyDeviceToHost, st));
  }
  CJT_CUDA_TRY(cudaStreamSynchronize(st));
  return CJT_OK;
}

int cjt_jacobi_shift(int32_t op, double alpha, double beta, const double* in, double* out,
                     int64_t n, int64_t batch, void* stream) {
  if (n < 0 || batch < 0 || (batch > 0 && (!in || !out))) return fail(CJT_EINVAL, "bad argument");
  if (batch > 65535 && (op == CJT_SHIFT_DEC_BETA || op == CJT_SHIFT_DEC_ALPHA))
    return fail(CJT_EINVAL, "decrement batch must be <= 65535 per call");
  const double ta = op == CJT_SHIFT_INC_ALPHA ? alpha + 1.0 : op == CJT_SHIFT_DEC_ALPHA ? alpha - 1.0 : alpha;
  const double tb = op == CJT_SHIFT_INC_BETA ? beta + 1.0 : op == CJT_SHIFT_DEC_BETA ? beta - 1.0 : beta;
  if (!(alpha > -1.0 && beta > -1.0 && ta > -1.0 && tb > -1.0))
    return fail(CJT_EINVAL, "inadmissible shift target: parameters must stay > -1");
  if (in == out && batch > 0) return fail(CJT_EINVAL, "in and out must not alias");
  return launch_shift(op, alpha, beta, in, out, n, batch, (cudaStream_t)stream);
}

int cjt_host_moments(double alpha, double beta, double mu0, int64_t g, double* mu) {
  if (g < 0 || !mu) return fail(CJT_EINVAL, "bad argument");
  // host code is compiled with -ffp-contract=off: every operation rounds as
  // in the reference's Python loop
  const double s = alpha + beta;
  mu[0] = mu0;
  if (g >= 1) mu[1] = (beta - alpha) / (s + 2.0) * mu0;
  const double two_d = 2.0 * (alpha - beta);
  for (int64_t k = 1; k < g; ++k) {
    const double kd = (double)k;
    mu[k + 1] = -(two_d * mu[k] + (s - kd + 2.0) * mu[k - 1]) / (s + kd + 2.0);
  }
  return CJT_OK;
}

int cjt_host_angles(const double* thetas, const int8_t* regions, int64_t n, double* x, double* xm) {
  if (n < 0 || (n > 0 && (!thetas || !regions || !x || !xm))) return fail(CJT_EINVAL, "null argument");
  for (int64_t i = 0; i < n; ++i) {
    const double th = thetas[i];
    x[i] = cos(th);
    if (regions[i] == 1) {
      const double h = sin(0.5 * th);
      xm[i] = -2.0 * h * h;
    } else if (regions[i] == -1) {
      const double h = cos(0.5 * th);
      xm[i] = 2.0 * h * h;
    } else {
      xm[i] = 0.0;
    }
  }
  return CJT_OK;
}

}  // extern "C"

// Device state of one backend-plugin call site (cjt_kernel_plan_*): the
// reference engine passes the same plan arrays on every forward / inverse
// (engine.py:177-183, 220-225), so tables, angles and the row layout are
// uploaded once and each call moves only its vector in and out.
struct cjt_kernel_plan {
  int kind = 0;                  // CJT_KERNEL_CLENSHAW / CJT_KERNEL_TRANSPOSE
  int device = 0;
  bool divide = false;           // clenshaw_smith (scalar API): divide by rb
  int64_t n_points = 0, n_len = 0, n_res = 0;
  std::vector<void*> allocs;
  RecTablesDev tab{};
  const double *rbp = nullptr, *rbm = nullptr, *rbpi = nullptr, *rbmi = nullptr;
  const double *x = nullptr, *xm = nullptr;
  const int8_t* reg = nullptr;
  const int64_t* cut = nullptr;
  double* d_in = nullptr;
  double* d_out = nullptr;
  std::unique_ptr<cjt_plan> P;   // transpose: single-vector inverse contraction plan
  double* d_ones = nullptr;
  std::vector<double> h_res;
  std::mutex mu;
  ~cjt_kernel_plan() {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    for (void* q : allocs) cudaFree(q);
    P.reset();
    cudaSetDevice(cur);
  }
};

namespace {

int kernel_plan_create(int32_t kind, const double* A, const double* B, const double* C, const double* r_plus,
                       const double* r_minus, const double* r_plus_inv, const double* r_minus_inv,
                       int64_t table_len, const double* thetas, const int64_t* cuts, const int8_t* regions,
                       int64_t n_points, int64_t n_len, bool divide, cjt_kernel_plan** out) {
  if (!out) return fail(CJT_EINVAL, "null argument");
  *out = nullptr;
  if (n_points < 0 || n_len < 0 || table_len < 0) return fail(CJT_EINVAL, "negative size");
  if (kind != CJT_KERNEL_CLENSHAW && kind != CJT_KERNEL_TRANSPOSE) return fail(CJT_EINVAL, "bad kernel kind");
  if (n_points > 0 && (!A || !B || !C || !r_plus || !r_minus || !r_plus_inv || !r_minus_inv || !thetas ||
                       !cuts || !regions))
    return fail(CJT_EINVAL, "null argument");
  int64_t maxcut = 0;
  for (int64_t i = 0; i < n_points; ++i) {
    if (cuts[i] < 0) return fail(CJT_EINVAL, "negative cut");
    maxcut = std::max(maxcut, cuts[i]);
  }
  if (maxcut > n_len)
    return fail(CJT_EINVAL, kind == CJT_KERNEL_CLENSHAW ? "cut exceeds the coefficient count"
                                                        : "cut exceeds the output length");
  std::unique_ptr<cjt_kernel_plan> K(new cjt_kernel_plan());
  CJT_CUDA_TRY(cudaGetDevice(&K->device));
  K->kind = kind;
  K->divide = divide;
  K->n_points = n_points;
  K->n_len = n_len;
  if (n_points == 0) {
    *out = K.release();
    return CJT_OK;
  }
  std::vector<double> x((size_t)n_points), xm((size_t)n_points);
  cjt_host_angles(thetas, regions, n_points, x.data(), xm.data());
  if (kind == CJT_KERNEL_CLENSHAW) {
    // C[n+1] is read up to n = maxcut - 1
    if (table_len < maxcut + 1) return fail(CJT_EINVAL, "recurrence tables are shorter than the largest cut + 1");
    const size_t tl = (size_t)maxcut + 1;
    double *dA, *dB, *dC, *rbp, *rbm, *rbpi, *rbmi, *dx, *dxm;
    int8_t* dreg;
    int64_t* dcut;
    const double* srcs[7] = {A, B, C, r_plus, r_minus, r_plus_inv, r_minus_inv};
    double** dsts[7] = {&dA, &dB, &dC, &rbp, &rbm, &rbpi, &rbmi};
    for (int k = 0; k < 7; ++k)
      if (int rc = upload(K->allocs, dsts[k], srcs[k], tl)) return rc;
    if (int rc = upload(K->allocs, &dx, x.data(), x.size())) return rc;
    if (int rc = upload(K->allocs, &dxm, xm.data(), xm.size())) return rc;
    if (int rc = upload(K->allocs, &dreg, regions, (size_t)n_points)) return rc;
    if (int rc = upload(K->allocs, &dcut, cuts, (size_t)n_points)) return rc;
    void* p;
    if (int rc = dalloc(K->allocs, &p, (size_t)std::max<int64_t>(n_len, 1) * 8)) return rc;
    K->d_in = (double*)p;
    if (int rc = dalloc(K->allocs, &p, (size_t)n_points * 8)) return rc;
    K->d_out = (double*)p;
    K->tab = RecTablesDev{dA, dB, dC, nullptr, nullptr, nullptr, nullptr, (int64_t)tl};
    K->rbp = rbp, K->rbm = rbm, K->rbpi = rbpi, K->rbmi = rbmi;
    K->x = dx, K->xm = dxm, K->reg = dreg, K->cut = dcut;
    CJT_CUDA_TRY(cudaDeviceSynchronize());
    *out = K.release();
    return CJT_OK;
  }
  if (table_len < maxcut) return fail(CJT_EINVAL, "tables shorter than the largest cut");
  // transpose: a single-vector inverse contraction plan over the caller's
  // rows, degrees 0..maxcut-1
  K->P.reset(new cjt_plan());
  cjt_plan* P = K->P.get();
  P->device = K->device;
  P->direction = CJT_INVERSE;
  P->n = std::max<int64_t>(maxcut, 1) - 1;
  P->G = n_points - 1;
  P->nrows = n_points;
  P->h_cut.assign(cuts, cuts + n_points);
  auto& Al = P->allocs;
  double *dx, *dxm;
  int8_t* dreg;
  int64_t* dcut;
  if (int rc = upload(Al, &dx, x.data(), x.size())) return rc;
  if (int rc = upload(Al, &dxm, xm.data(), xm.size())) return rc;
  if (int rc = upload(Al, &dreg, regions, (size_t)n_points)) return rc;
  if (int rc = upload(Al, &dcut, cuts, (size_t)n_points)) return rc;
  P->rows = RecRowsDev{dx, dxm, dreg, dcut, n_points};
  const size_t tl = (size_t)std::max<int64_t>(maxcut, 1);
  const double* src[7] = {A, B, C, r_plus, r_minus, r_plus_inv, r_minus_inv};
  if (int rc = upload_tables(Al, src, tl, &P->tab)) return rc;
  std::vector<int64_t> off((size_t)n_points);
  int64_t tot = 0;
  for (int64_t i = 0; i < n_points; ++i) {
    off[i] = tot;
    tot += (cuts[i] >= 1) ? (cuts[i] - 1) / CK : 0;
  }
  if (int rc = upload(Al, &P->ck_off, off.data(), off.size())) return rc;
  void* p;
  if (int rc = dalloc(Al, &p, (size_t)std::max<int64_t>(tot, 1) * sizeof(double2))) return rc;
  P->ck = (double2*)p;
  if (tot > 0)
    if (int rc = launch_checkpoints(P->rows, P->tab, P->ck_off, P->ck, 0)) return rc;
  if (int rc = reserve(P, 1)) return rc;
  K->n_res = P->n + 1;
  std::vector<double> ones((size_t)K->n_res, 1.0);
  if (int rc = upload(Al, &K->d_ones, ones.data(), ones.size())) return rc;
  if (int rc = dalloc(Al, &p, (size_t)n_points * 8)) return rc;
  K->d_in = (double*)p;
  if (int rc = dalloc(Al, &p, (size_t)K->n_res * 8)) return rc;
  K->d_out = (double*)p;
  K->h_res.resize((size_t)K->n_res);
  cjt_plan::Workspace* W = nullptr;
  if (int rc = get_workspace(P, 0, &W)) return rc;
  CJT_CUDA_TRY(cudaDeviceSynchronize());
  *out = K.release();
  return CJT_OK;
}

int kernel_plan_execute(cjt_kernel_plan* K, const double* in, double* out) {
  if (!K) return fail(CJT_EINVAL, "null plan");
  if (K->n_points == 0) return CJT_OK;
  if (!in || !out) return fail(CJT_EINVAL, "null buffer");
  DeviceGuard g(K->device);
  std::lock_guard<std::mutex> lk(K->mu);
  if (K->kind == CJT_KERNEL_CLENSHAW) {
    if (K->n_len > 0) CJT_CUDA_TRY(cudaMemcpy(K->d_in, in, (size_t)K->n_len * 8, cudaMemcpyHostToDevice));
    if (int rc = launch_clenshaw_points(K->tab, K->rbp, K->rbm, K->rbpi, K->rbmi, K->d_in, 0, K->x, K->xm,
                                        K->reg, K->cut, K->d_out, 0, K->n_points, 1, K->divide, 0))
      return rc;
    CJT_CUDA_TRY(cudaMemcpy(out, K->d_out, (size_t)K->n_points * 8, cudaMemcpyDeviceToHost));
    return CJT_OK;
  }
  cjt_plan* P = K->P.get();
  std::lock_guard<std::mutex> lp(P->exec_mu);
  cjt_plan::Workspace* W = nullptr;
  if (int rc = get_workspace(P, 0, &W)) return rc;
  CJT_CUDA_TRY(cudaMemcpy(K->d_in, in, (size_t)K->n_points * 8, cudaMemcpyHostToDevice));
  if (int rc = launch_rec_inverse(P->tab, P->inv_gen, P->nrows, P->iitems, P->n_iitems, P->tile_ids, K->d_in,
                                  K->n_points, 1, P->vt, false, P->G, W->part, 0))
    return rc;
  if (int rc = launch_inverse_finish(P->dt_slot0, P->dt_nslot, K->n_res, W->part, nullptr, K->d_ones, K->d_out,
                                     K->n_res, 1, 0))
    return rc;
  CJT_CUDA_TRY(cudaMemcpy(K->h_res.data(), K->d_out, (size_t)K->n_res * 8, cudaMemcpyDeviceToHost));
  for (int64_t k = 0; k < K->n_res && k < K->n_len; ++k) out[k] += K->h_res[(size_t)k];
  return CJT_OK;
}

int kernel_once(int32_t kind, const double* A, const double* B, const double* C, const double* rp,
                const double* rm, const double* rpi, const double* rmi, int64_t table_len, const double* thetas,
                const int64_t* cuts, const int8_t* regions, int64_t n_points, int64_t n_len, bool divide,
                const double* in, double* out) {
  cjt_kernel_plan* K = nullptr;
  if (int rc = kernel_plan_create(kind, A, B, C, rp, rm, rpi, rmi, table_len, thetas, cuts, regions, n_points,
                                  n_len, divide, &K))
    return rc;
  std::unique_ptr<cjt_kernel_plan> hold(K);
  return kernel_plan_execute(K, in, out);
}

}  // namespace

extern "C" {

int cjt_kernel_plan_create(int32_t kind, const double* A, const double* B, const double* C,
                           const double* r_plus, const double* r_minus, const double* r_plus_inv,
                           const double* r_minus_inv, int64_t table_len, const double* thetas,
                           const int64_t* cuts, const int8_t* regions, int64_t n_points, int64_t n_len,
                           cjt_kernel_plan** out) {
  return kernel_plan_create(kind, A, B, C, r_plus, r_minus, r_plus_inv, r_minus_inv, table_len, thetas, cuts,
                            regions, n_points, n_len, false, out);
}

int cjt_kernel_plan_execute(cjt_kernel_plan* plan, const double* in, double* out) {
  return kernel_plan_execute(plan, in, out);
}

int cjt_kernel_plan_destroy(cjt_kernel_plan* plan) {
  if (!plan) return CJT_OK;
  cudaDeviceSynchronize();
  delete plan;
  return CJT_OK;
}

int cjt_clenshaw_points(const double* A, const double* B, const double* C, const double* rb_plus,
                        const double* rb_minus, const double* rb_plus_inv, const double* rb_minus_inv,
                        const double* coeffs, int64_t n_coeffs, const double* thetas,
                        const int64_t* cuts, const int8_t* regions, double* out, int64_t n_points) {
  if (n_points < 0 || n_coeffs < 0) return fail(CJT_EINVAL, "negative size");
  int64_t maxcut = 0;
  for (int64_t i = 0; i < n_points; ++i) maxcut = std::max(maxcut, cuts[i]);
  return kernel_once(CJT_KERNEL_CLENSHAW, A, B, C, rb_plus, rb_minus, rb_plus_inv, rb_minus_inv, maxcut + 1,
                     thetas, cuts, regions, n_points, n_coeffs, false, coeffs, out);
}

int cjt_clenshaw_smith_points(const double* A, const double* B, const double* C, const double* rb_plus,
                              const double* rb_minus, const double* coeffs, int64_t n_coeffs,
                              const double* thetas, const int8_t* modes, int64_t n_points, double* out) {
  if (n_coeffs < 1 || n_points < 0) return fail(CJT_EINVAL, "need >= 1 coefficient");
  for (int64_t i = 0; i < n_points; ++i)
    if (modes[i] < -1 || modes[i] > 1) return fail(CJT_EINVAL, "mode must be -1, 0 or +1");
  std::vector<int64_t> cuts((size_t)n_points, n_coeffs);
  // the reciprocal tables are unused by the dividing variant
  return kernel_once(CJT_KERNEL_CLENSHAW, A, B, C, rb_plus, rb_minus, rb_plus, rb_minus, n_coeffs + 1, thetas,
                     cuts.data(), modes, n_points, n_coeffs, true, coeffs, out);
}

int cjt_clenshaw_points_dev(const double* A, const double* B, const double* C, const double* rb_plus,
                            const double* rb_minus, const double* rb_plus_inv,
                            const double* rb_minus_inv, int64_t table_len, const double* coeffs,
                            int64_t ldc, const double* x, const double* xm, const int64_t* cuts,
                            const int8_t* regions, double* out, int64_t ldo, int64_t n_points,
                            int64_t batch, void* stream) {
  if (n_points < 0 || batch < 0 || table_len < 0) return fail(CJT_EINVAL, "negative size");
  if (n_points == 0 || batch == 0) return CJT_OK;
  if (!A || !B || !C || !rb_plus || !rb_minus || !rb_plus_inv || !rb_minus_inv || !coeffs || !x ||
      !xm || !cuts || !regions || !out)
    return fail(CJT_EINVAL, "null argument");
  RecTablesDev tab{A, B, C, nullptr, nullptr, nullptr, nullptr, table_len};
  return launch_clenshaw_points(tab, rb_plus, rb_minus, rb_plus_inv, rb_minus_inv, coeffs, ldc, x, xm,
                                regions, cuts, out, ldo, n_points, batch, false, (cudaStream_t)stream);
}

int cjt_jacobi_values(const double* A, const double* B, const double* C, const double* rf_plus,
                      const double* rf_minus, int64_t table_len, int64_t n_max,
                      const double* thetas, const int8_t* modes, int64_t n_points, double* out) {
  if (n_points < 0 || n_max < 0) return fail(CJT_EINVAL, "negative size");
  if (n_points == 0) return CJT_OK;
  if (table_len < n_max) return fail(CJT_EINVAL, "tables shorter than n_max");
  for (int64_t i = 0; i < n_points; ++i)
    if (modes[i] < -1 || modes[i] > 1) return fail(CJT_EINVAL, "mode must be -1, 0 or +1");
  std::vector<double> x((size_t)n_points), xm((size_t)n_points);
  cjt_host_angles(thetas, modes, n_points, x.data(), xm.data());
  std::vector<void*> tmp;
  struct Free {
    std::vector<void*>* v;
    ~Free() { for (void* p : *v) cudaFree(p); }
  } fr{&tmp};
  const size_t tl = (size_t)std::max<int64_t>(n_max, 1);
  double *dA, *dB, *dC, *rfp, *rfm, *dx, *dxm;
  int8_t* dmode;
  const double* srcs[5] = {A, B, C, rf_plus, rf_minus};
  double** dsts[5] = {&dA, &dB, &dC, &rfp, &rfm};
  for (int k = 0; k < 5; ++k)
    if (int rc = upload(tmp, dsts[k], srcs[k], tl)) return rc;
  if (int rc = upload(tmp, &dx, x.data(), x.size())) return rc;
  if (int rc = upload(tmp, &dxm, xm.data(), xm.size())) return rc;
  if (int rc = upload(tmp, &dmode, modes, (size_t)n_points)) return rc;
  const size_t nout = (size_t)n_points * (size_t)(n_max + 1);
  void* p;
  if (int rc = dalloc(tmp, &p, nout * 8)) return rc;
  RecTablesDev tab{dA, dB, dC, rfp, rfm, nullptr, nullptr, (int64_t)tl};
  if (int rc = launch_jacobi_values(tab, n_max, dx, dxm, dmode, (double*)p, n_points, 0)) return rc;
  CJT_CUDA_TRY(cudaMemcpy(out, p, nout * 8, cudaMemcpyDeviceToHost));
  return CJT_OK;
}

int cjt_chirpz_create(const cjt_chirpz_desc* d, cjt_chirpz_plan** out) {
  if (!d || !out) return fail(CJT_EINVAL, "null argument");
  *out = nullptr;
  std::unique_ptr<cjt_chirpz_plan> C(new cjt_chirpz_plan());
  C->owner.reset(new cjt_plan());
  cjt_plan* P = C->owner.get();
  CJT_CUDA_TRY(cudaGetDevice(&P->device));
  {
    const double2* t = nullptr;
    if (int rc = shared_twiddles(8192, &t)) return rc;
    P->tw8192 = const_cast<double2*>(t);
  }
  if (int rc = build_chirpz(P, *d, &C->cz)) return rc;
  C->in_len = d->p0 + d->width;
  C->out_len = d->q0 - d->out_shift + d->count;
  CJT_CUDA_TRY(cudaDeviceSynchronize());
  *out = C.release();
  return CJT_OK;
}

int cjt_chirpz_execute(cjt_chirpz_plan* C, const double* in, int64_t ldi, double* out, int64_t ldo,
                       int64_t batch, void* stream) {
  if (!C) return fail(CJT_EINVAL, "null plan");
  if (batch < 0) return fail(CJT_EINVAL, "negative batch");
  if (batch == 0) return CJT_OK;
  if (!in || !out) return fail(CJT_EINVAL, "null buffer");
  if (ldi < C->in_len || ldo < C->out_len) return fail(CJT_EINVAL, "leading dimension too small");
  if (batch > 65535) return fail(CJT_EINVAL, "batch must be <= 65535 per call");
  DeviceGuard g(C->owner->device);
  cudaStream_t st = (cudaStream_t)stream;
  cjt_chirpz_plan::Ws* W = nullptr;
  {
    std::lock_guard<std::mutex> lk(C->mu);
    W = &C->ws[st];
    if (W->batch < batch) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(st, &cs);
      if (cs != cudaStreamCaptureStatusNone)
        return fail(CJT_EINVAL, "chirp-z workspace for this stream must exist before graph capture");
      for (void* q : W->allocs) cudaFree(q);
      *W = cjt_chirpz_plan::Ws{};
      void* p;
      const int64_t se = C->owner->scratch_elems_per_vec * batch;
      if (se > 0) {
        if (int rc = dalloc(W->allocs, &p, (size_t)se * 16)) return rc;
        W->scratch = (double2*)p;
      }
      int64_t pe = 0, spe = 0;
      chirpz_workspace(C->cz, batch, &pe, &spe);
      if (pe > 0) {
        if (int rc = dalloc(W->allocs, &p, (size_t)pe * 8)) return rc;
        W->part = (double*)p;
      }
      if (spe > 0) {
        if (int rc = dalloc(W->allocs, &p, (size_t)spe * 16)) return rc;
        W->spec = (double2*)p;
      }
      W->batch = batch;
    }
  }
  int launches = 0;
  return launch_chirpz(C->cz, C->owner->tw8192, in, ldi, out, ldo, batch, W->scratch, W->part, W->spec, st,
                       &launches);
}

int cjt_chirpz_destroy(cjt_chirpz_plan* C) {
  if (!C) return CJT_OK;
  cudaDeviceSynchronize();
  delete C;
  return CJT_OK;
}

int cjt_transpose_accumulate(const double* A, const double* B, const double* C, const double* rf_plus,
                             const double* rf_minus, const double* rf_plus_inv,
                             const double* rf_minus_inv, const double* wv, const double* thetas,
                             const int64_t* cuts, const int8_t* regions, double* out, int64_t n_out,
                             int64_t n_points, int64_t table_len) {
  return kernel_once(CJT_KERNEL_TRANSPOSE, A, B, C, rf_plus, rf_minus, rf_plus_inv, rf_minus_inv, table_len,
                     thetas, cuts, regions, n_points, n_out, false, wv, out);
}

}  // extern "C"
