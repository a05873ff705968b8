// ckg_api.cu — device context and the C-ABI (include/ckmpm_b200.h) of the
// B200-native CK-MPM transfer path.  Host orchestration of one substep in the
// reference's phase order (proj/include/ckmpm/simulation.hpp:150-188), one
// CUDA stream per context, no host round trip inside a substep.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../include/ckmpm_b200.h"
#include "ckg_bin.cuh"
#include "ckg_frame.cuh"
#include "ckg_io.cuh"
#include "ckg_isort.cuh"
#include "ckg_kernels.cuh"
#include "ckg_scan.cuh"
#include "ckg_slab.cuh"
#include "ckg_transfer.cuh"
#include "ckg_quad.cuh"
#include "ckg_g2p2g.cuh"

namespace ckg {
constexpr uint32_t kHostSmallSort = 2048;  // host-path crosser count sorted by one CTA

struct CudaError {
  cudaError_t e;
  const char* what;
};

namespace {

#define CKG_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) throw CudaError{_e, #call};   \
  } while (0)

struct ConfigFail {
  std::string msg;
};

template <typename T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

template <typename T>
T* dalloc(uint64_t count) {
  T* p = nullptr;
  if (count == 0) count = 1;
  CKG_CUDA(cudaMalloc(&p, count * sizeof(T)));
  return p;
}

int grid_for(uint64_t work, int threads, int max_blocks = 148 * 16) {
  uint64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > uint64_t(max_blocks)) b = max_blocks;
  return int(b);
}

const char* num_message(int code) {
  switch (code) {
    case CKG_NUM_FC_STRESS_INVERTED: return "fixed corotated stress: det F <= 0";
    case CKG_NUM_DP_STRESS_INVERTED: return "granular stress: det F <= 0";
    case CKG_NUM_FLUID_STATE_J: return "fluid state: J must be > 0";
    case CKG_NUM_NEAR_SINGULAR_D: return "near-singular APIC D matrix";
    case CKG_NUM_SINGULAR_MLS: return "singular MLS moment matrix";
    case CKG_NUM_RETURN_MAP_INVERTED: return "plastic return map: det F <= 0";
    case CKG_NUM_F_INVERTED: return "deformation gradient inverted";
    case CKG_NUM_FLUID_J: return "fluid compression drove J <= 0";
    case CKG_NUM_INACTIVE_BLOCK: return "access to inactive grid block";
    default: return "numerical error";
  }
}

}  // namespace

// Precision-independent interface of a context.
struct CtxBase {
  ckg_config cfg{};
  std::string last_error;
  uint64_t step_count = 0;  // substeps completed (for the non-finite message)
  virtual ~CtxBase() = default;
  virtual int upload(const void* p, uint64_t n) = 0;
  virtual int download(void* p, uint64_t n) = 0;
  virtual uint64_t count() const = 0;
  virtual int step(double dt, int stop_after, int count, ckg_step_out* out) = 0;
  virtual int advance_frame(const ckg_frame_in* in, ckg_frame_out* out) = 0;
  virtual uint64_t record_bytes(int kind) const = 0;
  virtual int pack_records(int kind, void* host, uint64_t bytes, int async) = 0;
  virtual int records_wait() = 0;
  virtual int debug_sort(uint32_t* keys, uint32_t* order, uint64_t n) = 0;
  virtual int debug_bases(int32_t* bases, uint64_t n) = 0;
  virtual uint64_t active_blocks() = 0;
  virtual bool is_fused() const = 0;
  virtual void* stream() const = 0;
  virtual int grid_download(int32_t* coords, double* nodes, uint64_t nb) = 0;
  virtual int grid_totals(double* mass, double* mom) = 0;
  virtual int diagnostics(ckg_diagnostics* out) = 0;
  virtual int slab_set(int rank, int world, int lo, int hi) = 0;
  virtual int slab_rebound(int lo, int hi) = 0;
  virtual int slab_plane_counts(uint64_t* counts) = 0;
  virtual int slab_bin(double dt, void* core_out) = 0;
  virtual int slab_p2g(const void* core_in, uint64_t* plane_blocks, int part) = 0;
  virtual int slab_halo(int op, int plane, void* buf) = 0;
  virtual int slab_grid() = 0;
  virtual int slab_g2p(uint64_t* counts) = 0;
  virtual int slab_pack(uint64_t nl_in, void* left, void* right) = 0;
  virtual int slab_finish(const void* left, uint64_t nl, const void* right, uint64_t nr, ckg_step_out* out) = 0;
  virtual int timer_mark(int slot) = 0;
  virtual int timer_elapsed(int a, int b, double* ms) = 0;
};

template <typename T>
struct Context final : CtxBase {
  int device = 0;
  cudaStream_t st = nullptr;
  // activation (dilate / directory scan / compaction) forked onto st_act after
  // the key pass, concurrent with the incremental sort on st (joined by
  // enqueue_activate): it needs only the footprint flags
  cudaStream_t st_act = nullptr;
  cudaEvent_t ev_key = nullptr, ev_act = nullptr;
  bool act_pre = false;
  bool clear_pre = false;  // the pool clear went with the forked activation
  cudaEvent_t ev[8] = {};  // phase boundaries; ev[7]: before a fused substep's deferred clear
  cudaEvent_t tev[16] = {};
  uint64_t launches = 0;  // kernels enqueued by the current API call
  uint64_t n = 0;
  int D = 0;
  uint64_t nd = 0;  // D^3
  int key_bits = 1;
  // particles (double-buffered SoA)
  T* fbuf[2] = {nullptr, nullptr};
  uint32_t* mbuf[2] = {nullptr, nullptr};
  T* tbuf[2] = {nullptr, nullptr};  // stress cache (6 x n) per state buffer
  bool stress_valid = false;
  int cur = 0;
  uint64_t cap = 0;  // particle buffer capacity (field stride)
  uint64_t wb[2] = {0, 0};  // window base of each state buffer (slab mode: room to prepend migrants)
  // x-slab decomposition (ckg_slab.cuh)
  bool slab = false;
  int srank = 0, sworld = 1, bx_lo = 0, bx_hi = 0;
  int pend_lo = -1, pend_hi = -1;  // rebalanced bounds, effective from this substep's migration
  uint32_t* plane_start = nullptr;
  uint32_t *fl_stay = nullptr, *fl_left = nullptr, *fl_right = nullptr;
  uint32_t *pos_stay = nullptr, *pos_left = nullptr, *pos_right = nullptr;
  uint64_t mig_left = 0, mig_right = 0, n_stay = 0;
  // region path of the migration (ckg_slab.cuh): sorted prefix [0, PL) and
  // suffix [PR, n) hold every possible crosser; mig_region = false falls back
  // to relaying out the whole slab
  bool mig_region = false;
  uint64_t reg_pl = 0, reg_pr = 0, stay_l = 0, stay_r = 0;
  unsigned long long* dreg = nullptr;  // PL, PR, far count
  double slab_dt = 0;
  // staging for AoS transfers
  T* staging = nullptr;
  uint64_t staging_words = 0;
  // sort
  uint32_t* keys = nullptr;
  uint32_t* vals = nullptr;
  RadixScratch rs;
  uint32_t* perm = nullptr;  // sorted position -> current index (result of the last sort)
  uint32_t* skeys = nullptr; // sorted keys
  // incremental sort state (ckg_isort.cuh)
  uint32_t* ko = nullptr;    // sorted keys of the stored order (valid after a completed step)
  bool ko_valid = false;
  uint32_t *chg = nullptr, *cpre = nullptr, *ck = nullptr, *ci = nullptr, *iota = nullptr;
  uint32_t *perm_buf = nullptr, *skeys_tmp = nullptr, *ncount = nullptr;
  uint32_t* wcnt = nullptr;  // changed count per warp of stored positions (chg holds the ballot words, cpre their scan)
  uint32_t* hcount = nullptr;  // pinned
  uint64_t last_changed = 0;
  int last_sort_kind = 0;    // 0 full radix, 1 identity, 2 incremental
  // grid
  uint32_t* core = nullptr;   // footprint blocks (D^3)
  uint32_t* flags = nullptr;  // active = dilated core (D^3)
  uint32_t* seg_begin = nullptr;
  uint32_t* seg_end = nullptr;
  int p2g_ctas = 0, g2p_ctas = 0;
  int p2gq_ctas = 0, g2pq_ctas = 0;  // quadratic baseline kernels
  int32_t* dir = nullptr;
  uint32_t* active = nullptr;
  uint32_t* rec = nullptr;   // per-item transfer records (kRecWords per active slot)
  uint32_t* cord = nullptr;  // P2G class order of every chunk (sorted positions)
  uint4* ccnt = nullptr;     // class counts of chunks past a segment's first
  uint8_t* cls8 = nullptr;   // P2G class per particle (state order), from the key pass
  uint32_t* scan_partials = nullptr;
  uint32_t* scan_partials_n = nullptr;  // scan scratch sized for n
  T* pool = nullptr;
  uint32_t pool_cap = 0;
  // fused G2P2G mode (ckg_g2p2g.cuh): two dense block pools
  // (slot = block key).  dpool[pa] holds the next substep's P2G when
  // pend_valid (scattered by the last fused kernel with dt pend_dt), else
  // zero; dpool[pa ^ 1] holds the last substep's grid over the active list
  // when defer_clear (kept for the grid facade, cleared at the next substep),
  // else zero.  pools_dirty: contents unknown (upload, failure).
  bool fused = false;
  T* dpool[2] = {nullptr, nullptr};
  int pa = 0;
  bool pend_valid = false, defer_clear = false, pools_dirty = true;
  double pend_dt = 0;
  int fused_ctas = 0;
  uint32_t* act_alt = nullptr;  // the previous substep's active list (fused mode)
  // deterministic mode (cfg.deterministic; det_gather_kernel): per active
  // block P2G tiles summed in a fixed order, out-of-tile records applied in
  // particle order.  Single domain only.
  bool det = false;
  T* dtile = nullptr;
  uint32_t dcap = 0;
  DetSpill<T>* dspill = nullptr;
  DetBuf<T> detbuf() const {
    // (the quadratic baseline's P2G keeps its atomic flush)
    if (!det || quad()) return DetBuf<T>{nullptr, 0u, nullptr, 0u};
    return DetBuf<T>{dtile, dcap, dspill, uint32_t(kDetSpillMax)};
  }
  void set_det_cap(uint32_t c) {
    dfree(dtile);
    dcap = c;
    dtile = dalloc<T>(uint64_t(c) * kDetVals);
  }
  T* facade_pool = nullptr;  // pool the grid facade reads (fused mode)
  // status
  DevStatus* dstat = nullptr;
  DevStatus* hstat = nullptr;  // pinned
  BcParam<T>* dbcs = nullptr;
  double* dacc = nullptr;  // diagnostics accumulators (11)
  uint64_t last_active = 0;
  bool grid_valid = false;
  // device frame driver (ckg_frame.cuh): one instantiated graph per starting
  // state buffer, rebuilt when anything baked into it changes
  FrameState* dframe = nullptr;
  FrameState* hframe = nullptr;  // pinned
  T* ddt = nullptr;
  uint32_t* dnc = nullptr;
  // capture streams: conditional bodies (0..2) and the two substeps'
  // forked activations (3, 4), with their fork / join events
  cudaStream_t cst[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t gev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaGraphExec_t fexec[2] = {nullptr, nullptr};
  struct GraphKey {
    uint64_t n = ~0ull, cap = 0;
    const void *pool = nullptr, *f0 = nullptr, *f1 = nullptr, *ko = nullptr;
    double mass_eps = 0;
    uint32_t pool_cap = 0;
    bool operator==(const GraphKey& o) const {
      return n == o.n && cap == o.cap && pool == o.pool && f0 == o.f0 && f1 == o.f1 && ko == o.ko &&
             mass_eps == o.mass_eps && pool_cap == o.pool_cap;
    }
  } fkey[2];
  uint64_t graph_kernels = 0;  // kernels per graph substep (both sort branches counted once each)
  // checkpoint / snapshot records (ckg_io.cuh): packed on the context stream,
  // copied to the host on their own stream so later substeps overlap the D2H
  uint32_t* iobuf = nullptr;
  uint64_t iobuf_words = 0;
  cudaStream_t iost = nullptr;
  cudaEvent_t io_packed = nullptr, io_done = nullptr;
  bool io_pending = false;

  explicit Context(const ckg_config& c) {
    cfg = c;
    device = c.device;
    CKG_CUDA(cudaSetDevice(device));
    CKG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CKG_CUDA(cudaStreamCreateWithFlags(&st_act, cudaStreamNonBlocking));
    CKG_CUDA(cudaEventCreateWithFlags(&ev_key, cudaEventDisableTiming));
    CKG_CUDA(cudaEventCreateWithFlags(&ev_act, cudaEventDisableTiming));
    for (auto& e : ev) CKG_CUDA(cudaEventCreate(&e));
    for (auto& e : tev) CKG_CUDA(cudaEventCreate(&e));
    D = c.resolution / 4 + 2;
    nd = uint64_t(D) * D * D;
    key_bits = 1;
    while ((uint64_t(1) << key_bits) < nd) ++key_bits;
    flags = dalloc<uint32_t>(nd);
    CKG_CUDA(cudaMemset(flags, 0, nd * sizeof(uint32_t)));
    core = dalloc<uint32_t>(nd);
    CKG_CUDA(cudaMemset(core, 0, nd * sizeof(uint32_t)));
    seg_begin = dalloc<uint32_t>(nd);
    seg_end = dalloc<uint32_t>(nd);
    CKG_CUDA(cudaMemset(seg_begin, 0, nd * sizeof(uint32_t)));
    CKG_CUDA(cudaMemset(seg_end, 0, nd * sizeof(uint32_t)));
    setup_persistent();
    dir = dalloc<int32_t>(nd);
    CKG_CUDA(cudaMemset(dir, 0xff, nd * sizeof(int32_t)));
    scan_partials = dalloc<uint32_t>(scan_tiles(std::max<uint64_t>(nd, 1)) + 1);
    // Block pool: the dense bound (every directory slot active) when it fits
    // in 16 GiB, so no substep can overflow; otherwise grown on demand.
    uint64_t dense_bytes = nd * kBlockVals * sizeof(T);
    uint64_t cap = dense_bytes <= (16ull << 30) ? nd : std::min<uint64_t>(nd, 1u << 16);
    set_pool_cap(uint32_t(cap));
    dstat = dalloc<DevStatus>(1);
    CKG_CUDA(cudaMemset(dstat, 0, sizeof(DevStatus)));
    status_reset_kernel<<<1, 32, 0, st>>>(dstat, 1, 1);
    CKG_CUDA(cudaMallocHost(&hstat, sizeof(DevStatus)));
    std::memset(hstat, 0, sizeof(DevStatus));
    dbcs = dalloc<BcParam<T>>(kMaxBoundaries);
    std::vector<BcParam<T>> hb(kMaxBoundaries);
    for (int b = 0; b < c.n_boundaries; ++b) {
      const ckg_boundary& s = c.boundaries[b];
      BcParam<T>& d = hb[b];
      d.kind = s.kind;
      for (int a = 0; a < 3; ++a) {
        d.lo[a] = T(s.lo[a]);
        d.hi[a] = T(s.hi[a]);
        d.normal[a] = T(s.normal[a]);
        d.velocity[a] = T(s.velocity[a]);
        d.omega[a] = T(s.omega[a]);
        d.center[a] = T(s.center[a]);
      }
    }
    CKG_CUDA(cudaMemcpy(dbcs, hb.data(), sizeof(BcParam<T>) * kMaxBoundaries, cudaMemcpyHostToDevice));
    dacc = dalloc<double>(12);
    if (c.deterministic) {
      det = true;
      set_det_cap(std::min<uint32_t>(pool_cap, 1u << 16));
      dspill = dalloc<DetSpill<T>>(kDetSpillMax);
    }
    // fused G2P2G (opt-in: CKG_FLAG_FUSED or CKMPM_FUSED=1)
    const char* fe = std::getenv("CKMPM_FUSED");
    if (((fe && fe[0] == '1') || (cfg.flags & CKG_FLAG_FUSED)) && fused_supported()) enable_fused();
  }

  bool is_fused() const override { return fused; }
  void* stream() const override { return static_cast<void*>(st); }

  bool fused_supported() const {
    return !quad() && cfg.scheme != CKG_SCHEME_MLS && !slab && !det && pool_cap >= nd;
  }

  template <int S, int MM>
  void fused_attr(int& per) {
    const size_t smem = g2p2g_smem_bytes<T, S>();
    CKG_CUDA(cudaFuncSetAttribute(g2p2g_kernel<T, S, MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    CKG_CUDA(cudaFuncSetAttribute(g2p2g_kernel<T, S, MM>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int p = 0;
    CKG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p, g2p2g_kernel<T, S, MM>, kFThreads, smem));
    per = per == 0 ? p : std::min(per, p);
  }

  void enable_fused() {
    if (fused) return;
    dpool[0] = pool;
    dpool[1] = dalloc<T>(uint64_t(nd) * kBlockVals);
    act_alt = dalloc<uint32_t>(pool_cap);
    pa = 0;
    pend_valid = defer_clear = false;
    pools_dirty = true;
    int nsm = 0, per = 0;
    CKG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    if (cfg.scheme == CKG_SCHEME_PIC) {
      fused_attr<kSchemePic, kMFC>(per);
      fused_attr<kSchemePic, kMDP>(per);
      fused_attr<kSchemePic, kMAll>(per);
    } else {
      fused_attr<kSchemeApic, kMFC>(per);
      fused_attr<kSchemeApic, kMDP>(per);
      fused_attr<kSchemeApic, kMAll>(per);
    }
    fused_ctas = std::max(1, per) * nsm;
    fused = true;
  }

  // Back to one compacted pool (slab mode): the dense pools' contents are dropped.
  void disable_fused() {
    if (!fused) return;
    CKG_CUDA(cudaStreamSynchronize(st));
    pool = dpool[0];
    dfree(dpool[1]);
    dfree(act_alt);
    dpool[0] = nullptr;
    fused = false;
    pend_valid = defer_clear = false;
    CKG_CUDA(cudaMemset(pool, 0, uint64_t(pool_cap) * kBlockVals * sizeof(T)));
  }

  ~Context() override {
    cudaSetDevice(device);
    if (st) cudaStreamSynchronize(st);
    for (int b = 0; b < 2; ++b) {
      dfree(fbuf[b]);
      dfree(mbuf[b]);
      dfree(tbuf[b]);
    }
    if (iost) cudaStreamSynchronize(iost);
    dfree(iobuf);
    if (io_packed) cudaEventDestroy(io_packed);
    if (io_done) cudaEventDestroy(io_done);
    if (iost) cudaStreamDestroy(iost);
    for (auto& e : fexec)
      if (e) cudaGraphExecDestroy(e);
    for (auto& c : cst)
      if (c) cudaStreamDestroy(c);
    for (auto& e : gev)
      if (e) cudaEventDestroy(e);
    dfree(dframe);
    dfree(ddt);
    dfree(dnc);
    if (hframe) cudaFreeHost(hframe);
    dfree(staging);
    dfree(keys);
    dfree(vals);
    dfree(rs.keys_alt);
    dfree(rs.vals_alt);
    dfree(rs.hist);
    dfree(rs.partials);
    for (uint32_t** b : {&ko, &chg, &cpre, &ck, &ci, &iota, &perm_buf, &skeys_tmp, &ncount, &wcnt}) dfree(*b);
    for (uint32_t** b : {&plane_start, &fl_stay, &fl_left, &fl_right, &pos_stay, &pos_left, &pos_right}) dfree(*b);
    dfree(dreg);
    if (hcount) cudaFreeHost(hcount);
    dfree(flags);
    dfree(core);
    dfree(seg_begin);
    dfree(seg_end);
    dfree(dir);
    dfree(active);
    dfree(rec);
    dfree(cord);
    dfree(ccnt);
    dfree(cls8);
    dfree(scan_partials);
    dfree(scan_partials_n);
    if (fused) {
      dfree(dpool[1]);
      dfree(act_alt);
    }
    dfree(dtile);
    dfree(dspill);
    dfree(pool);
    dfree(dstat);
    dfree(dbcs);
    dfree(dacc);
    if (hstat) cudaFreeHost(hstat);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : tev)
      if (e) cudaEventDestroy(e);
    if (ev_key) cudaEventDestroy(ev_key);
    if (ev_act) cudaEventDestroy(ev_act);
    if (st_act) cudaStreamDestroy(st_act);
    if (st) cudaStreamDestroy(st);
  }

  void set_pool_cap(uint32_t cap) {
    dfree(pool);
    dfree(active);
    dfree(rec);
    pool_cap = cap;
    pool = dalloc<T>(uint64_t(cap) * kBlockVals);
    active = dalloc<uint32_t>(cap);
    rec = dalloc<uint32_t>(uint64_t(cap) * kRecWords);
  }

  PState<T> state(int b) const { return PState<T>{fbuf[b] + wb[b], mbuf[b] + wb[b], tbuf[b] + wb[b], n, cap}; }
  PState<T> state_at(int b, uint64_t base, uint64_t count) const {
    return PState<T>{fbuf[b] + base, mbuf[b] + base, tbuf[b] + base, count, cap};
  }

  // Smallest shared-memory carveout holding two CTAs of a P2G kernel: the
  // rest of the 256 KB stays L1 for the class-order particle gathers and spills.
  template <typename K>
  void set_two_cta_carveout(K* kernel, size_t smem, int ctas = 2) {
    cudaFuncAttributes fa{};
    CKG_CUDA(cudaFuncGetAttributes(&fa, kernel));
    int smem_sm = 0;
    CKG_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device));
    const size_t need = size_t(ctas) * (smem + fa.sharedSizeBytes + 1024);  // + 1 KB reserved per CTA
    // supported sm_100 carveouts (KB); the driver rounds the percentage up to
    // the next one, so ask for floor(target) of the smallest that fits
    size_t target = size_t(smem_sm);
    for (int kb : {64, 100, 132, 164, 196, 228})
      if (size_t(kb) * 1024 >= need) {
        target = std::min<size_t>(size_t(kb) * 1024, size_t(smem_sm));
        break;
      }
    const int pct = int(std::min<size_t>(100, target * 100 / std::max(smem_sm, 1)));
    CKG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
  }

  template <typename K>
  void g2p_attr(K* kernel) {
    CKG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(g2p_dyn_smem<T>())));
  }

  template <int S>
  void occupancy_for() {
    int nsm = 0, per = 0;
    CKG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    const size_t smem = p2g_smem_bytes<T>();
    CKG_CUDA(cudaFuncSetAttribute(p2g_tile_kernel<T, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    set_two_cta_carveout(p2g_tile_kernel<T, S, true>, smem,
                         p2g_min_ctas<T>());
    CKG_CUDA(cudaFuncSetAttribute(p2g_tile_kernel<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    set_two_cta_carveout(p2g_tile_kernel<T, S>, smem,
                         p2g_min_ctas<T>());
    CKG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, p2g_tile_kernel<T, S>, kP2GThreads, smem));
    if (cfg.scheme == S) p2g_ctas = std::max(1, per) * nsm;
    g2p_attr(g2p_tile_kernel<T, S, 0, kMFC>);
    g2p_attr(g2p_tile_kernel<T, S, 0, kMDP>);
    g2p_attr(g2p_tile_kernel<T, S>);
    CKG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, g2p_tile_kernel<T, S>, kG2PThreads, g2p_dyn_smem<T>()));
    if (cfg.scheme == S) g2p_ctas = std::max(1, per) * nsm;
    if constexpr (S != kSchemeMls) {
      if (quad() && cfg.scheme == S) {
        const size_t qs = p2g_quad_smem_bytes<T>();
        CKG_CUDA(cudaFuncSetAttribute(p2g_quad_kernel<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(qs)));
        set_two_cta_carveout(p2g_quad_kernel<T, S>, qs, quad_min_ctas<T>());
        CKG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, p2g_quad_kernel<T, S>, kQThreads, qs));
        p2gq_ctas = std::max(1, per) * nsm;
        g2p_attr(g2p_tile_kernel<T, S, 1>);
        CKG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, g2p_tile_kernel<T, S, 1>, kG2PThreads,
                                                               g2p_dyn_smem<T>()));
        g2pq_ctas = std::max(1, per) * nsm;
      }
    }
  }

  void setup_persistent() {
    occupancy_for<kSchemePic>();
    occupancy_for<kSchemeApic>();
    occupancy_for<kSchemeMls>();
  }

  void ensure_particles(uint64_t count) {
    // slab mode keeps headroom for migrants (the particle count of a rank changes)
    const uint64_t want = slab ? count + std::max<uint64_t>(count / 2, 1u << 20) : count;
    if (fbuf[0] && want <= cap && (slab || count == cap)) {
      n = count;
      wb[0] = wb[1] = slab ? (cap - count) / 2 : 0;
      return;
    }
    for (int b = 0; b < 2; ++b) {
      dfree(fbuf[b]);
      dfree(mbuf[b]);
      dfree(tbuf[b]);
    }
    dfree(keys);
    dfree(vals);
    dfree(rs.keys_alt);
    dfree(rs.vals_alt);
    dfree(rs.hist);
    dfree(rs.partials);
    for (uint32_t** b : {&ko, &chg, &cpre, &ck, &ci, &iota, &perm_buf, &skeys_tmp, &ncount, &wcnt}) dfree(*b);
    n = count;
    cap = std::max<uint64_t>(want, 1);
    wb[0] = wb[1] = slab ? (cap - count) / 2 : 0;
    for (int b = 0; b < 2; ++b) {
      fbuf[b] = dalloc<T>(uint64_t(kNumFields) * cap);
      mbuf[b] = dalloc<uint32_t>(cap);
      tbuf[b] = dalloc<T>(6 * cap);
    }
    keys = dalloc<uint32_t>(cap);
    vals = dalloc<uint32_t>(cap);
    dfree(cord);
    dfree(ccnt);
    dfree(cls8);
    cls8 = dalloc<uint8_t>(cap);
    cord = dalloc<uint32_t>(cap);
    ccnt = dalloc<uint4>(cap / kP2GChunk + 2);
    rs.keys_alt = dalloc<uint32_t>(cap);
    rs.vals_alt = dalloc<uint32_t>(cap);
    uint64_t nh = uint64_t(kRadix) * sort_tiles(cap);
    rs.hist = dalloc<uint32_t>(nh);
    rs.partials = dalloc<uint32_t>(scan_tiles(nh) + 1);
    for (uint32_t** b : {&ko, &chg, &cpre, &ck, &ci, &iota, &perm_buf, &skeys_tmp}) *b = dalloc<uint32_t>(cap);
    ncount = dalloc<uint32_t>(1);
    wcnt = dalloc<uint32_t>(cap / 32 + 1);
    dfree(scan_partials_n);
    scan_partials_n = dalloc<uint32_t>(scan_tiles(cap) + 1);
    if (!hcount) CKG_CUDA(cudaMallocHost(&hcount, sizeof(uint32_t)));
    iota_kernel<<<grid_for(cap, 256, 1 << 30), 256, 0, st>>>(iota, cap);
    if (slab) {
      for (uint32_t** b : {&fl_stay, &fl_left, &fl_right, &pos_stay, &pos_left, &pos_right}) {
        dfree(*b);
        *b = dalloc<uint32_t>(cap);
      }
    }
    ko_valid = false;
    cur = 0;
  }

  void ensure_staging(uint64_t words) {
    if (staging_words >= words) return;
    dfree(staging);
    staging = dalloc<T>(words);
    staging_words = words;
  }

  int upload(const void* p, uint64_t count) override {
    CKG_CUDA(cudaSetDevice(device));
    ensure_particles(count);
    if (count == 0) return CKG_OK;
    const uint64_t words = count * (kNumFields + 1);
    ensure_staging(words);
    CKG_CUDA(cudaMemcpyAsync(staging, p, words * sizeof(T), cudaMemcpyHostToDevice, st));
    aos_to_soa_kernel<T><<<grid_for(count, kXpTile, 148 * 16), 256, 0, st>>>(staging, state(cur));
    CKG_CUDA(cudaGetLastError());
    CKG_CUDA(cudaStreamSynchronize(st));
    grid_valid = false;
    stress_valid = false;
    ko_valid = false;
    pend_valid = defer_clear = false;
    pools_dirty = true;
    return CKG_OK;
  }

  int download(void* p, uint64_t count) override {
    if (count != n) {
      last_error = "download: particle count mismatch";
      return CKG_ERR_CONFIG;
    }
    if (count == 0) return CKG_OK;
    CKG_CUDA(cudaSetDevice(device));
    const uint64_t words = count * (kNumFields + 1);
    ensure_staging(words);
    soa_to_aos_kernel<T><<<grid_for(count, kXpTile, 148 * 16), 256, 0, st>>>(state(cur), staging);
    CKG_CUDA(cudaGetLastError());
    CKG_CUDA(cudaMemcpyAsync(p, staging, words * sizeof(T), cudaMemcpyDeviceToHost, st));
    CKG_CUDA(cudaStreamSynchronize(st));
    return CKG_OK;
  }

  uint64_t count() const override { return n; }

  int quad() const { return (cfg.flags & CKG_FLAG_QUADRATIC) ? 1 : 0; }

  StepConst<T> make_const(double dt) const {
    StepConst<T> c{};
    c.quad = quad();
    c.dense = fused ? 1 : 0;
    c.dx = T(cfg.dx);
    c.inv_dx = T(cfg.inv_dx);
    c.dt = T(dt);
    c.mass_eps = T(cfg.mass_eps);
    c.clamp_floor = T(cfg.clamp_floor);
    for (int a = 0; a < 3; ++a) c.gravity[a] = T(cfg.gravity[a]);
    c.res = cfg.resolution;
    c.D = D;
    c.scheme = cfg.scheme;
    c.n_materials = cfg.n_materials;
    c.clamp_singular = cfg.clamp_singular;
    c.n_boundaries = cfg.n_boundaries;
    {
      // power-of-two dx: x/dx is exactly x*inv_dx (same exact scaling)
      int e = 0;
      const double fr = std::frexp(cfg.dx, &e);
      c.pow2 = (fr == 0.5 && cfg.inv_dx * cfg.dx == 1.0) ? 1 : 0;
    }
    for (int m = 0; m < cfg.n_materials && m < kMaxMaterials; ++m) {
      const ckg_material& s = cfg.materials[m];
      MatParam<T>& d = c.mats[m];
      d.model = s.model;
      d.mu = T(s.mu);
      d.lambda = T(s.lambda);
      d.dp_alpha = T(s.dp_alpha);
      d.bulk = T(s.bulk);
      d.gamma = T(s.gamma);
      d.viscosity = T(s.viscosity);
      d.density = T(s.density);
    }
    return c;
  }

  // K1 + K2: key/footprint pass then stable sort (perm[i] = source index of
  // sorted position i, skeys[i] its key).  With the stored order's sorted
  // keys at hand the sort is incremental (ckg_isort.cuh); one small host
  // read-back of the changed count picks identity / merge / full radix.
  void enqueue_sort(bool pre_activate = false, bool pre_clear = false) {
    PState<T> cs = state(cur);
    if (act_pre) {  // a forked activation never joined (an abandoned substep)
      CKG_CUDA(cudaStreamWaitEvent(st, ev_act, 0));
      act_pre = false;
    }
    (quad() ? key_footprint_kernel<T, 1> : key_footprint_kernel<T, 0>)
        <<<grid_for((n + kKeyPer - 1) / kKeyPer, 256, 1 << 30), 256, 0, st>>>(
        cs, T(cfg.inv_dx), cfg.resolution, D, quad(), keys, core, ko_valid ? ko : nullptr, chg, wcnt, quad() ? nullptr : cls8, dstat);
    launches += 1;
    if (pre_activate) fork_activate(pre_clear);
    if (ko_valid) {
      CKG_CUDA(cudaMemcpyAsync(hcount, &dstat->nchanged, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
      CKG_CUDA(cudaStreamSynchronize(st));
      const uint32_t nc = *hcount;
      last_changed = nc;
      if (nc != 0 && uint64_t(nc) * 8 <= n) {
        exclusive_scan(wcnt, cpre, (n + 31) / 32, scan_partials_n, st);
        compact_changed_kernel<<<grid_for((n + 31) / 32, 256, 1 << 30), 256, 0, st>>>(keys, chg, cpre, n, ck, ci);
        launches += 4;
      }
      if (nc == 0) {
        perm = iota;
        skeys = ko;
        last_sort_kind = 1;
        return;
      }
      if (uint64_t(nc) * 8 <= n) {
        uint32_t *sck = nullptr, *sci = nullptr;
        if (nc <= kHostSmallSort) {
          // a few crossers: one-CTA bitonic sort (one launch instead of the
          // radix passes)
          static bool attr = false;
          if (!attr) {
            CKG_CUDA(cudaFuncSetAttribute(small_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(kSmallSort * sizeof(unsigned long long))));
            attr = true;
          }
          uint32_t m = 1;
          while (m < nc) m <<= 1;
          sck = rs.keys_alt;
          sci = rs.vals_alt;
          small_sort_kernel<<<1, 1024, m * sizeof(unsigned long long), st>>>(ck, ci, &dstat->nchanged, sck, sci);
          launches += 1;
        } else {
          radix_sort_pairs(ck, ci, nc, key_bits, rs, st, &sck, &sci, ci);
          launches += uint64_t((key_bits + kRadixBits - 1) / kRadixBits) * 5;
        }
        const uint64_t tiles = (n + kMergeTile - 1) / kMergeTile;
        merge_bounds_kernel<<<grid_for(tiles, 256, 1 << 30), 256, 0, st>>>(keys, chg, n, sck, sci, nc, nullptr,
                                                                           wcnt);
        merge_unchanged_kernel<<<unsigned((n + 256 * kMergePer - 1) / (256 * kMergePer)), 256, 0, st>>>(keys, chg, cpre, n, sck, sci, nc, nullptr,
                                                                       wcnt, perm_buf, skeys_tmp);
        // seg_begin/end still hold the previous substep's runs of ko unless
        // the stored order was rebuilt since (slab migration)
        const bool segs = !slab;
        merge_changed_kernel<<<grid_for(nc, 256, 1 << 30), 256, 0, st>>>(
            ko, chg, cpre, n, sck, sci, nc, nullptr, segs ? seg_begin : nullptr, segs ? seg_end : nullptr, perm_buf,
            skeys_tmp);
        launches += 3;
        std::swap(ko, skeys_tmp);
        perm = perm_buf;
        skeys = ko;
        last_sort_kind = 2;
        return;
      }
    }
    uint32_t *sk = nullptr, *sp = nullptr;
    radix_sort_pairs(keys, vals, n, key_bits, rs, st, &sk, &sp);
    launches += uint64_t((key_bits + kRadixBits - 1) / kRadixBits) * 5;
    CKG_CUDA(cudaMemcpyAsync(ko, sk, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    perm = sp;
    skeys = ko;
    ko_valid = true;
    last_sort_kind = 0;
    last_changed = n;
  }

  // K3-K6: inset error in sorted order, halo dilation, directory, segments.
  // The part of the activation that needs only the footprint flags: halo
  // dilation, directory scan, compaction into the active list.
  void enqueue_activate_flags(cudaStream_t s) {
    dilate_kernel<<<grid_for(nd, 256, 1 << 30), 256, 0, s>>>(core, flags, D);
    exclusive_scan(flags, reinterpret_cast<uint32_t*>(dir), nd, scan_partials, s);
    if (slab)
      plane_start_kernel<<<(D + 1 + 127) / 128, 128, 0, s>>>(reinterpret_cast<const uint32_t*>(dir), flags, D,
                                                            plane_start);
    // (the segment table is reset on st below: the sort may still read it)
    compact_kernel<<<grid_for(nd, 256, 1 << 30), 256, 0, s>>>(core, flags, dir, active, nullptr, nullptr, nd,
                                                              pool_cap, dstat);
    if (slab) slab_ranges_kernel<<<1, 1, 0, s>>>(plane_start, D, bx_lo, bx_hi, dstat);
  }
  // Fork the flag-only activation (and, with_clear, the pool clear, which
  // needs only the new active list) after the key pass just enqueued on st.
  void fork_activate(bool with_clear) {
    CKG_CUDA(cudaEventRecord(ev_key, st));
    CKG_CUDA(cudaStreamWaitEvent(st_act, ev_key, 0));
    enqueue_activate_flags(st_act);
    if (with_clear) clear_kernel<T><<<148 * 8, 256, 0, st_act>>>(pool, dstat, pool_cap);
    clear_pre = with_clear;
    CKG_CUDA(cudaEventRecord(ev_act, st_act));
    act_pre = true;
  }

  void enqueue_activate(int step_idx, bool want_cord = true) {
    PState<T> cs = state(cur);
    if (act_pre) {
      CKG_CUDA(cudaStreamWaitEvent(st, ev_act, 0));
      act_pre = false;
    } else {
      enqueue_activate_flags(st);
    }
    CKG_CUDA(cudaMemsetAsync(seg_begin, 0, nd * sizeof(uint32_t), st));
    CKG_CUDA(cudaMemsetAsync(seg_end, 0, nd * sizeof(uint32_t), st));
    inset_fixup_kernel<T><<<148, 256, 0, st>>>(cs, perm, T(cfg.inv_dx), cfg.resolution, dstat, step_idx);
    segments_kernel<<<grid_for((n + 3) / 4, 256, 1 << 30), 256, 0, st>>>(skeys, n, seg_begin, seg_end);
    xfer_prep_kernel<T><<<148 * 8, kPrepWarps * 32, 0, st>>>(cs, perm, make_const(0.0), dir, active, seg_begin, seg_end,
                                                 pool_cap, dstat, rec, cord, ccnt,
                                                 (quad() || !want_cord) ? nullptr : cls8);
  }

  template <int S>
  void enqueue_p2g(const StepConst<T>& c, int step_idx) {
    if (quad()) {
      if constexpr (S != kSchemeMls)
        p2g_quad_kernel<T, S><<<p2gq_ctas, kQThreads, p2g_quad_smem_bytes<T>(), st>>>(
            state(cur), perm, c, dir, active, seg_begin, seg_end, pool, pool_cap, dstat, step_idx);
      return;
    }
    const DetBuf<T> db = detbuf();
    (db.tile ? p2g_tile_kernel<T, S, true> : p2g_tile_kernel<T, S, false>)
        <<<p2g_ctas, kP2GThreads, p2g_smem_bytes<T>(), st>>>(state(cur), perm, c, dir, rec, cord, ccnt, pool,
                                                              pool_cap, dstat, step_idx, db);
    // deterministic mode: the fixed-order tile sums (x-slab ranks first
    // exchange their boundary planes' tiles: slab_grid runs the gather)
    if (db.tile && !slab) enqueue_det_gather();
  }
  template <int S>
  void enqueue_g2p(const StepConst<T>& c, int step_idx) {
    if (quad()) {
      if constexpr (S != kSchemeMls)
        g2p_tile_kernel<T, S, 1><<<g2pq_ctas, kG2PThreads, g2p_dyn_smem<T>(), st>>>(state(cur), state(cur ^ 1), perm, c, dir,
                                                                     rec, pool, pool_cap, dstat, step_idx);
      return;
    }
    // narrowest material-model instance covering the scene
    int mm = cfg.clamp_singular ? kMClamp : 0;
    for (int m = 0; m < cfg.n_materials; ++m)
      mm |= cfg.materials[m].model == kModelFC ? kMFC : cfg.materials[m].model == kModelDP ? kMDP : kMFluid;
    if (mm == kMFC || mm == 0)
      g2p_tile_kernel<T, S, 0, kMFC><<<g2p_ctas, kG2PThreads, g2p_dyn_smem<T>(), st>>>(state(cur), state(cur ^ 1), perm, c, dir,
                                                                       rec, pool, pool_cap, dstat, step_idx);
    else if (mm == kMDP)
      g2p_tile_kernel<T, S, 0, kMDP><<<g2p_ctas, kG2PThreads, g2p_dyn_smem<T>(), st>>>(state(cur), state(cur ^ 1), perm, c, dir,
                                                                       rec, pool, pool_cap, dstat, step_idx);
    else
      g2p_tile_kernel<T, S><<<g2p_ctas, kG2PThreads, g2p_dyn_smem<T>(), st>>>(state(cur), state(cur ^ 1), perm, c, dir, rec, pool,
                                                                pool_cap, dstat, step_idx);
  }

  void enqueue_det_gather() {
    const DetBuf<T> db = detbuf();
    det_gather_kernel<T><<<148 * 8, 256, 0, st>>>(pool, active, dir, db.tile, db.cap, dstat, pool_cap, D);
    det_spill_kernel<T><<<1, 1024, 0, st>>>(pool, dir, db.spill, dstat, pool_cap, D, slab ? 1 : 0);
    launches += 2;
  }

  // Kernels enqueue_step launches (status reset, key/footprint, 5 per radix
  // pass, inset fix-up, dilate, 3-kernel scan, compact, segments, clear,
  // P2G, grid, G2P).
  uint64_t launches_per_step(int stop_after) const {
    uint64_t k = 1;  // status reset; sort kernels are counted by enqueue_sort
    if (stop_after >= CKG_PHASE_ACTIVATE) k += 8;
    if (stop_after >= CKG_PHASE_CLEAR) k += 1;
    if (stop_after >= CKG_PHASE_P2G) k += 1;
    if (stop_after >= CKG_PHASE_GRID) k += 1;
    if (stop_after >= CKG_PHASE_G2P) k += 1;
    return k;
  }

  // Enqueue one substep up to stop_after; errors are latched on the device.
  void enqueue_step(double dt, int stop_after, int step_idx, bool reset_err, bool timed) {
    const StepConst<T> c = make_const(dt);
    launches += launches_per_step(stop_after);
    status_reset_kernel<<<1, 32, 0, st>>>(dstat, reset_err ? 1 : 0);
    if (timed) CKG_CUDA(cudaEventRecord(ev[0], st));
    // (deterministic mode: the tile gather writes every node of the active blocks)
    const bool want_clear = stop_after >= CKG_PHASE_CLEAR && !detbuf().tile;
    enqueue_sort(stop_after >= CKG_PHASE_ACTIVATE && !slab, want_clear);
    if (timed) CKG_CUDA(cudaEventRecord(ev[1], st));
    if (stop_after >= CKG_PHASE_ACTIVATE) enqueue_activate(step_idx);
    if (timed) CKG_CUDA(cudaEventRecord(ev[2], st));
    if (want_clear && !clear_pre) clear_kernel<T><<<148 * 8, 256, 0, st>>>(pool, dstat, pool_cap);
    clear_pre = false;
    if (timed) CKG_CUDA(cudaEventRecord(ev[3], st));
    if (stop_after >= CKG_PHASE_P2G) {
      if (!stress_valid) {
        stress_kernel<T><<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(state(cur), perm, c, dstat, step_idx);
        stress_valid = true;
        launches += 1;
      }
      if (cfg.scheme == CKG_SCHEME_PIC) enqueue_p2g<kSchemePic>(c, step_idx);
      else if (cfg.scheme == CKG_SCHEME_APIC) enqueue_p2g<kSchemeApic>(c, step_idx);
      else enqueue_p2g<kSchemeMls>(c, step_idx);
    }
    if (timed) CKG_CUDA(cudaEventRecord(ev[4], st));
    if (stop_after >= CKG_PHASE_GRID)
      grid_update_kernel<T><<<148 * 8, 256, 0, st>>>(pool, active, dstat, pool_cap, c, dbcs);
    if (timed) CKG_CUDA(cudaEventRecord(ev[5], st));
    if (stop_after >= CKG_PHASE_G2P) {
      if (cfg.scheme == CKG_SCHEME_PIC) enqueue_g2p<kSchemePic>(c, step_idx);
      else if (cfg.scheme == CKG_SCHEME_APIC) enqueue_g2p<kSchemeApic>(c, step_idx);
      else enqueue_g2p<kSchemeMls>(c, step_idx);
    }
    if (timed) CKG_CUDA(cudaEventRecord(ev[6], st));
    CKG_CUDA(cudaGetLastError());
  }

  // ---------------------------------------------------------------- fused G2P2G
  template <int S>
  void enqueue_fused_kernel(const StepConst<T>& c, double dt_next, int step_idx) {
    int mm = cfg.clamp_singular ? kMClamp : 0;
    for (int m = 0; m < cfg.n_materials; ++m)
      mm |= cfg.materials[m].model == kModelFC ? kMFC : cfg.materials[m].model == kModelDP ? kMDP : kMFluid;
    const size_t smem = g2p2g_smem_bytes<T, S>();
    T* in = dpool[pa];
    T* out = dpool[pa ^ 1];
    if (mm == kMFC || mm == 0)
      g2p2g_kernel<T, S, kMFC><<<fused_ctas, kFThreads, smem, st>>>(state(cur), state(cur ^ 1), perm, c, rec,
                                                                      pool_cap, in, out, T(dt_next), dstat, step_idx);
    else if (mm == kMDP)
      g2p2g_kernel<T, S, kMDP><<<fused_ctas, kFThreads, smem, st>>>(state(cur), state(cur ^ 1), perm, c, rec,
                                                                      pool_cap, in, out, T(dt_next), dstat, step_idx);
    else
      g2p2g_kernel<T, S, kMAll><<<fused_ctas, kFThreads, smem, st>>>(state(cur), state(cur ^ 1), perm, c, rec,
                                                                       pool_cap, in, out, T(dt_next), dstat, step_idx);
  }

  // One substep in fused mode up to stop_after.  The P2G of
  // this substep is normally already in dpool[pa] (scattered by the previous
  // substep's fused kernel with the same dt); otherwise the plain P2G runs.
  // A full substep ends with the fused kernel: G2P of this substep from
  // dpool[pa], P2G of the next one into dpool[pa ^ 1] at the same dt.
  void enqueue_fused_step(double dt, int stop_after, bool timed) {
    const StepConst<T> c = make_const(dt);
    const uint64_t pool_bytes = uint64_t(pool_cap) * kBlockVals * sizeof(T);
    if (pools_dirty) {
      CKG_CUDA(cudaMemsetAsync(dpool[0], 0, pool_bytes, st));
      CKG_CUDA(cudaMemsetAsync(dpool[1], 0, pool_bytes, st));
      pools_dirty = pend_valid = defer_clear = false;
    }
    // the last substep's grid (kept for the facade) is cleared over its
    // active list right before the fused kernel scatters into that pool
    // (L2-resident when the kernel's reductions arrive); its list is kept
    // while this substep's activation builds the new one
    const bool clear_prev = defer_clear;
    if (clear_prev) std::swap(active, act_alt);
    defer_clear = false;
    const bool need_p2g = !pend_valid || pend_dt != dt;
    launches += 1;
    status_reset_kernel<<<1, 32, 0, st>>>(dstat, 1, need_p2g ? 1 : 0);
    if (timed) CKG_CUDA(cudaEventRecord(ev[0], st));
    enqueue_sort(stop_after >= CKG_PHASE_ACTIVATE && !slab);
    if (timed) CKG_CUDA(cudaEventRecord(ev[1], st));
    if (stop_after >= CKG_PHASE_ACTIVATE) {
      enqueue_activate(0, need_p2g);
      launches += 8;
    }
    if (timed) CKG_CUDA(cudaEventRecord(ev[2], st));
    if (stop_after >= CKG_PHASE_CLEAR && need_p2g && pend_valid) {
      // a speculative scatter at another dt: its footprint lies in this
      // substep's active set
      clear_list_kernel<T><<<148 * 8, 256, 0, st>>>(dpool[pa], active, &dstat->n_active, pool_cap);
      launches += 1;
    }
    if (timed) CKG_CUDA(cudaEventRecord(ev[3], st));
    if (stop_after >= CKG_PHASE_P2G) {
      pool = dpool[pa];
      if (need_p2g) {
        if (!stress_valid) {
          stress_kernel<T><<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(state(cur), perm, c, dstat, 0);
          stress_valid = true;
          launches += 1;
        }
        if (cfg.scheme == CKG_SCHEME_PIC) enqueue_p2g<kSchemePic>(c, 0);
        else enqueue_p2g<kSchemeApic>(c, 0);
      } else {
        promote_pending_error_kernel<<<1, 32, 0, st>>>(dstat);
      }
      launches += 1;
    }
    if (timed) CKG_CUDA(cudaEventRecord(ev[4], st));
    if (stop_after >= CKG_PHASE_GRID) {
      grid_update_kernel<T><<<148 * 8, 256, 0, st>>>(dpool[pa], active, dstat, pool_cap, c, dbcs);
      launches += 1;
    }
    if (timed) CKG_CUDA(cudaEventRecord(ev[5], st));
    if (stop_after >= CKG_PHASE_G2P && clear_prev) {
      clear_list_kernel<T><<<148 * 8, 256, 0, st>>>(dpool[pa ^ 1], act_alt, &dstat->n_active_prev, pool_cap);
      launches += 1;
    }
    if (timed) CKG_CUDA(cudaEventRecord(ev[7], st));
    if (stop_after >= CKG_PHASE_G2P) {
      if (cfg.scheme == CKG_SCHEME_PIC) enqueue_fused_kernel<kSchemePic>(c, dt, 0);
      else enqueue_fused_kernel<kSchemeApic>(c, dt, 0);
      launches += 1;
    }
    if (timed) CKG_CUDA(cudaEventRecord(ev[6], st));
    CKG_CUDA(cudaGetLastError());
  }

  // Host bookkeeping after a fused-mode call (rc: its status).
  void fused_after(int stop_after, int rc) {
    if (rc == CKG_OK && stop_after >= CKG_PHASE_G2P) {
      facade_pool = dpool[pa];  // this substep's grid (kept until the next substep)
      pa ^= 1;
      pend_valid = true;
      pend_dt = last_dt;
      defer_clear = true;
      stress_valid = false;  // the fused kernel writes no stress cache
    } else {
      facade_pool = dpool[pa];
      pools_dirty = true;
      pend_valid = defer_clear = false;
    }
    pool = facade_pool;
  }
  double last_dt = 0;

  void fill_out(ckg_step_out* out, bool timed, int stop_after) {
    std::memset(out, 0, sizeof(*out));
    const DevStatus& h = *hstat;
    double vm2 = 0;
    unsigned long long vb = h.vmax2;
    std::memcpy(&vm2, &vb, sizeof vm2);
    out->vmax = double(std::sqrt(T(vm2)));
    for (int m = 0; m < CKG_MAX_MATERIALS; ++m) {
      double j;
      unsigned long long b = h.minj[m];
      std::memcpy(&j, &b, sizeof j);
      out->min_j[m] = std::isfinite(j) ? j : 1.0;
    }
    // node visits per particle (TransferCounters, transfer.hpp:32-45): the
    // compact kernel's 2 x 8 dual-grid nodes (MLS scatters them twice), the
    // quadratic baseline's 27 (transfer.hpp:285-320, :512-543)
    const uint64_t per = quad() ? 27 : cfg.scheme == CKG_SCHEME_MLS ? 32 : 16;
    const uint64_t per_g = quad() ? 27 : 16;
    if (stop_after >= CKG_PHASE_P2G) {
      out->p2g_node_visits = per * n;
      out->p2g_transfers = n;
    }
    if (stop_after >= CKG_PHASE_G2P) {
      out->g2p_node_visits = per_g * n;
      out->g2p_transfers = n;
    }
    out->active_blocks = h.n_active;
    if (timed) {
      for (int k = 0; k < 6; ++k) {
        float ms = 0;
        cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
        out->phase_ms[k] = ms;
      }
      if (fused && stop_after >= CKG_PHASE_G2P) {
        // fused: the last substep's grid is cleared between the grid update
        // (ev[5]) and the fused kernel (ev[7] .. ev[6])
        float ms = 0;
        cudaEventElapsedTime(&ms, ev[5], ev[7]);
        out->phase_ms[2] += ms;
        cudaEventElapsedTime(&ms, ev[7], ev[6]);
        out->phase_ms[5] = ms;
      }
    }
  }

  // Returns CKG status; fills out.
  int decode_status(ckg_step_out* out, int stop_after) {
    const DevStatus& h = *hstat;
    if (h.err != ~0ull) {
      const unsigned long long p = h.err;
      const int code = int(p & 0xff);
      const int axis = int((p >> 8) & 0xf);
      const uint64_t particle = (p >> 12) & 0xffffffffffull;
      const int phase = int((p >> 52) & 0xf);
      out->status = CKG_ERR_NUMERICAL;
      out->error_code = code;
      out->error_axis = axis;
      out->error_particle = particle;
      out->error_phase = phase;
      char buf[256];
      if (code == CKG_NUM_OUT_OF_DOMAIN)
        std::snprintf(buf, sizeof buf, "particle %llu violates the 2-cell domain inset on axis %d",
                      (unsigned long long)particle, axis);
      else
        std::snprintf(buf, sizeof buf, "%s", num_message(code));
      last_error = buf;
      return CKG_ERR_NUMERICAL;
    }
    if (stop_after >= CKG_PHASE_G2P && h.nonfinite) {
      out->status = CKG_ERR_NUMERICAL;
      out->error_code = CKG_NUM_NONFINITE;
      out->error_phase = CKG_PHASE_G2P;
      last_error = "non-finite particle state after step " + std::to_string(step_count + 1);
      return CKG_ERR_NUMERICAL;
    }
    return CKG_OK;
  }

  int step(double dt, int stop_after, int count_steps, ckg_step_out* out) override {
    CKG_CUDA(cudaSetDevice(device));
    ckg_step_out local;
    if (!out) out = &local;
    if (n == 0) {
      std::memset(out, 0, sizeof(*out));
      for (double& j : out->min_j) j = 1.0;
      if (stop_after >= CKG_PHASE_G2P) step_count += uint64_t(count_steps);
      out->substeps_done = stop_after >= CKG_PHASE_G2P ? uint64_t(count_steps) : 0;
      return CKG_OK;
    }
    if (count_steps == 1) return step_one(dt, stop_after, true, out);
    // several full substeps at one dt with the frame graph in its fixed-dt
    // mode: no host round trip between substeps (the sort path is chosen on
    // the device); it stops at a failing substep like the loop below
    if (stop_after >= CKG_PHASE_G2P && graph_ready()) return graph_steps(dt, count_steps, out);
    // several substeps: one at a time, so a failing substep leaves the state
    // of the last completed one and a pool overflow grows the pool and
    // retries (every substep already waits for its key pass's changed count,
    // so nothing is lost by checking the status in between)
    uint64_t total_launches = 0;
    int rc = CKG_OK;
    uint64_t done = 0;
    for (int k = 0; k < count_steps; ++k) {
      rc = step_one(dt, CKG_PHASE_G2P, false, out);
      total_launches += out->kernel_launches;
      if (rc != CKG_OK) break;
      ++done;
    }
    out->kernel_launches = total_launches;
    out->substeps_done = done;
    return rc;
  }

  // count substeps at fixed dt through the frame graph (graph_ready()).
  int graph_steps(double dt, int count, ckg_step_out* out) {
    const int c0 = cur;
    if (!fexec[c0] || !(fkey[c0] == graph_key())) build_frame_graph(c0);
    FrameState fs{};
    fs.fixed_dt = double(T(dt));
    fs.target = uint32_t(count);
    fs.max_substeps = uint32_t(count);
    fs.frame_dt = 1.0;
    fs.frame_end = 0.0;
    fs.vmax = 0.0;
    for (int m = 0; m < kMaxMaterials; ++m) fs.min_j[m] = 1.0;
    fs.parity = uint32_t(cur);
    *hframe = fs;
    CKG_CUDA(cudaMemcpyAsync(dframe, hframe, sizeof(FrameState), cudaMemcpyHostToDevice, st));
    CKG_CUDA(cudaGraphLaunch(fexec[c0], st));
    CKG_CUDA(cudaMemcpyAsync(hframe, dframe, sizeof(FrameState), cudaMemcpyDeviceToHost, st));
    CKG_CUDA(cudaMemcpyAsync(hstat, dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
    CKG_CUDA(cudaStreamSynchronize(st));
    const uint32_t done = hframe->substeps;
    const bool failed = hframe->status == 2;
    cur = int(hframe->parity);
    step_count += done;
    perm = perm_buf;
    skeys = ko;
    grid_valid = true;
    last_active = hstat->n_active;
    fill_out(out, false, CKG_PHASE_G2P);
    out->kernel_launches = uint64_t(done + (failed ? 1 : 0)) * graph_kernels;
    out->substeps_done = done;
    if (!failed) {
      out->status = CKG_OK;
      return CKG_OK;
    }
    ko_valid = false;  // the failing substep re-sorted; the stored order did not move
    if (hstat->overflow) {
      last_error = "grid block pool capacity exceeded";
      out->status = CKG_ERR_DEVICE;
      return CKG_ERR_DEVICE;
    }
    const int rc = decode_status(out, CKG_PHASE_G2P);
    out->status = rc;
    return rc;
  }

  // One substep up to stop_after (timed: per-phase device events).
  int step_one(double dt, int stop_after, bool timed, ckg_step_out* out) {
    launches = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
      if (fused) {
        last_dt = dt;
        enqueue_fused_step(dt, stop_after, timed);
      } else {
        enqueue_step(dt, stop_after, 0, true, timed);
      }
      CKG_CUDA(cudaMemcpyAsync(hstat, dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
      CKG_CUDA(cudaStreamSynchronize(st));
      if ((hstat->overflow & 3u) && !fused) {
        ko_valid = false;
        // grow the pool / the deterministic tile buffer (state untouched:
        // G2P writes the other buffer)
        const uint64_t want = std::min<uint64_t>(nd, uint64_t(hstat->n_active) * 5 / 4 + 64);
        if (hstat->overflow & 1u) set_pool_cap(uint32_t(want));
        if (hstat->overflow & 2u) set_det_cap(uint32_t(std::min<uint64_t>(want, pool_cap)));
        continue;
      }
      break;
    }
    fill_out(out, timed, stop_after);
    out->kernel_launches = launches;
    out->sort_changed = last_changed;
    out->sort_kind = last_sort_kind;
    out->substeps_done = 0;
    grid_valid = true;
    last_active = hstat->n_active;
    if (hstat->overflow & 4u) {
      last_error = "deterministic mode: more than 4096 out-of-tile particles in one substep";
      out->status = CKG_ERR_DEVICE;
      return CKG_ERR_DEVICE;
    }
    if (hstat->overflow) {
      last_error = "grid block pool capacity exceeded";
      out->status = CKG_ERR_DEVICE;
      return CKG_ERR_DEVICE;
    }
    int rc = decode_status(out, stop_after);
    if (fused) fused_after(stop_after, rc);
    if (rc == CKG_OK && stop_after >= CKG_PHASE_G2P) {
      cur ^= 1;
      step_count += 1;
      out->substeps_done = 1;
    } else {
      ko_valid = false;  // stored order unchanged: the new sorted keys do not describe it
    }
    if (stop_after < CKG_PHASE_ACTIVATE) CKG_CUDA(cudaMemsetAsync(core, 0, nd * sizeof(uint32_t), st));
    out->status = rc;
    return rc;
  }

  // ---------------------------------------------------------------- frame driver
  // cfl_dt (simulation.hpp:134-145) on the host, in T, for the substeps the
  // graph does not run (first substep after an upload, host-loop fallback).
  T host_cfl_dt(const FrameState& fs, T remaining) const {
    T cmax = T(0);
    for (int mi = 0; mi < cfg.n_materials && mi < kMaxMaterials; ++mi) {
      const ckg_material& m = cfg.materials[mi];
      T sp;
      if (m.model == CKG_MODEL_J_FLUID)
        sp = std::sqrt(T(m.bulk) * T(m.gamma) * std::pow(T(fs.min_j[mi]), T(1) - T(m.gamma)) / T(m.density));
      else
        sp = std::sqrt((T(m.lambda) + T(2) * T(m.mu)) / T(m.density));
      cmax = std::max(cmax, sp);
    }
    const T denom = std::max(T(fs.vmax), cmax);
    T dt = denom > T(0) ? T(fs.cfl) * T(cfg.dx) / denom : remaining;
    if (T(fs.max_dt) > T(0)) dt = std::min(dt, T(fs.max_dt));
    return std::min(dt, remaining);
  }

  static cudaGraph_t capture_graph_of(cudaStream_t s) {
    cudaStreamCaptureStatus cs;
    unsigned long long id;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CKG_CUDA(cudaStreamGetCaptureInfo(s, &cs, &id, &g, &deps, &nd));
    return g;
  }
  // Appends a conditional node after the capture's current tail; the stream
  // continues after it. Returns the (first) body graph.
  static cudaGraph_t add_conditional(cudaStream_t s, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type) {
    cudaStreamCaptureStatus cs;
    unsigned long long id;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CKG_CUDA(cudaStreamGetCaptureInfo(s, &cs, &id, &g, &deps, &nd));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = type;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    CKG_CUDA(cudaGraphAddNode(&node, g, deps, nd, &p));
    CKG_CUDA(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
    return p.conditional.phGraph_out[0];
  }

  // One substep of the frame graph, captured on `s` (conditional sort bodies
  // on `s_aux`), reading and writing state buffer `cs` -> cs ^ 1.
  void capture_graph_substep(cudaStream_t s, cudaStream_t s_aux, int cs, cudaGraphConditionalHandle h_loop,
                             cudaGraphConditionalHandle h_next, cudaStream_t s_fork, cudaEvent_t e_key,
                             cudaEvent_t e_act) {
    const cudaStream_t saved_st = st, saved_fork = st_act;
    const cudaEvent_t saved_key = ev_key, saved_act = ev_act;
    const int saved_cur = cur;
    st = s;
    cur = cs;
    // the activation forked off the sort as in the host loop (fork_activate)
    st_act = s_fork;
    ev_key = e_key;
    ev_act = e_act;
    StepConst<T> c = make_const(0.0);
    c.dtp = ddt;
    uint64_t k = 0;
    frame_ctl_kernel<T><<<1, 32, 0, st>>>(dframe, c, ddt);
    status_reset_kernel<<<1, 32, 0, st>>>(dstat, 1);
    // sort: crossers counted on the device; <= kSmallSort of them are merged
    // into the stored order, more take the full radix (IF nodes)
    (quad() ? key_footprint_kernel<T, 1> : key_footprint_kernel<T, 0>)
        <<<grid_for((n + kKeyPer - 1) / kKeyPer, 256, 1 << 30), 256, 0, st>>>(
        state(cur), T(cfg.inv_dx), cfg.resolution, D, quad(), keys, core, ko, chg, wcnt, quad() ? nullptr : cls8, dstat);
    fork_activate(true);
    const uint64_t nw = (n + 31) / 32;
    exclusive_scan(wcnt, cpre, nw, scan_partials_n, st);
    compact_changed_kernel<<<grid_for((n + 31) / 32, 256, 1 << 30), 256, 0, st>>>(keys, chg, cpre, n, ck, ci);
    k += 7;
    cudaGraph_t g = capture_graph_of(st);
    cudaGraphConditionalHandle hs, hm, hf;
    CKG_CUDA(cudaGraphConditionalHandleCreate(&hs, g, 0, cudaGraphCondAssignDefault));
    CKG_CUDA(cudaGraphConditionalHandleCreate(&hm, g, 0, cudaGraphCondAssignDefault));
    CKG_CUDA(cudaGraphConditionalHandleCreate(&hf, g, 0, cudaGraphCondAssignDefault));
    const uint32_t bound = uint32_t(std::max<uint64_t>(n / 8, kSmallSort));
    sort_decide_kernel<<<1, 32, 0, st>>>(cpre, wcnt, nw, bound, dnc, dframe, hs, hm, hf);
    k += 1;
    const uint64_t tiles = (n + kMergeTile - 1) / kMergeTile;
    // crossers sorted into (sck, sci): merge them with the stored order
    auto merge = [&](cudaStream_t s2, uint32_t* sck, uint32_t* sci, uint32_t max_nc) {
      merge_bounds_kernel<<<grid_for(tiles, 256, 1 << 30), 256, 0, s2>>>(keys, chg, n, sck, sci, 0u, dnc, wcnt);
      merge_unchanged_kernel<<<unsigned((n + 256 * kMergePer - 1) / (256 * kMergePer)), 256, 0, s2>>>(keys, chg, cpre, n, sck, sci, 0u, dnc, wcnt,
                                                                      perm_buf, skeys_tmp);
      merge_changed_kernel<<<grid_for(max_nc, 256, 1 << 30), 256, 0, s2>>>(ko, chg, cpre, n, sck, sci, 0u, dnc,
                                                                           seg_begin, seg_end, perm_buf, skeys_tmp);
      CKG_CUDA(cudaMemcpyAsync(ko, skeys_tmp, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s2));
    };
    {
      cudaGraph_t body = add_conditional(st, hm, cudaGraphCondTypeIf);
      CKG_CUDA(cudaStreamBeginCaptureToGraph(s_aux, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
      const uint32_t pad_key = key_bits >= 32 ? 0xffffffffu : uint32_t((1ull << key_bits) - 1);
      pad_crossers_kernel<<<grid_for(bound, 256), 256, 0, s_aux>>>(ck, ci, dnc, bound, pad_key);
      uint32_t *sck = nullptr, *sci = nullptr;
      radix_sort_pairs(ck, ci, bound, key_bits, rs, s_aux, &sck, &sci, ci);
      merge(s_aux, sck, sci, bound);
      cudaGraph_t done;
      CKG_CUDA(cudaStreamEndCapture(s_aux, &done));
    }
    {
      cudaGraph_t body = add_conditional(st, hs, cudaGraphCondTypeIf);
      CKG_CUDA(cudaStreamBeginCaptureToGraph(s_aux, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
      uint32_t *sck = rs.keys_alt, *sci = rs.vals_alt;
      small_sort_kernel<<<1, 1024, kSmallSort * sizeof(unsigned long long), s_aux>>>(ck, ci, dnc, sck, sci);
      merge(s_aux, sck, sci, kSmallSort);
      cudaGraph_t done;
      CKG_CUDA(cudaStreamEndCapture(s_aux, &done));
      k += 4;
    }
    {
      cudaGraph_t body = add_conditional(st, hf, cudaGraphCondTypeIf);
      CKG_CUDA(cudaStreamBeginCaptureToGraph(s_aux, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
      uint32_t *sk = nullptr, *sp = nullptr;
      radix_sort_pairs(keys, vals, n, key_bits, rs, s_aux, &sk, &sp);
      CKG_CUDA(cudaMemcpyAsync(ko, sk, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s_aux));
      CKG_CUDA(cudaMemcpyAsync(perm_buf, sp, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s_aux));
      cudaGraph_t done;
      CKG_CUDA(cudaStreamEndCapture(s_aux, &done));
    }
    perm = perm_buf;
    skeys = ko;
    enqueue_activate(0);  // (joins the forked activation and clear)
    if (!clear_pre) clear_kernel<T><<<148 * 8, 256, 0, st>>>(pool, dstat, pool_cap);
    clear_pre = false;
    if (cfg.scheme == CKG_SCHEME_PIC) enqueue_p2g<kSchemePic>(c, 0);
    else if (cfg.scheme == CKG_SCHEME_APIC) enqueue_p2g<kSchemeApic>(c, 0);
    else enqueue_p2g<kSchemeMls>(c, 0);
    grid_update_kernel<T><<<148 * 8, 256, 0, st>>>(pool, active, dstat, pool_cap, c, dbcs);
    if (cfg.scheme == CKG_SCHEME_PIC) enqueue_g2p<kSchemePic>(c, 0);
    else if (cfg.scheme == CKG_SCHEME_APIC) enqueue_g2p<kSchemeApic>(c, 0);
    else enqueue_g2p<kSchemeMls>(c, 0);
    frame_end_kernel<T><<<1, 32, 0, st>>>(dframe, dstat, h_loop, h_next, cfg.n_materials);
    k += 8 + 1 + 3 + 1;
    graph_kernels = k;
    CKG_CUDA(cudaGetLastError());
    st = saved_st;
    cur = saved_cur;
    st_act = saved_fork;
    ev_key = saved_key;
    ev_act = saved_act;
  }

  GraphKey graph_key() const {
    GraphKey k;
    k.n = n;
    k.cap = cap;
    k.pool = pool;
    k.f0 = fbuf[0];
    k.f1 = fbuf[1];
    k.ko = ko;
    k.mass_eps = cfg.mass_eps;
    k.pool_cap = pool_cap;
    return k;
  }

  // WHILE(h_loop) { substep(c0 -> c0^1); IF(h_next) { substep(c0^1 -> c0) } }
  void build_frame_graph(int c0) {
    if (!dframe) {
      dframe = dalloc<FrameState>(1);
      ddt = dalloc<T>(1);
      dnc = dalloc<uint32_t>(1);
      CKG_CUDA(cudaMallocHost(&hframe, sizeof(FrameState)));
      for (auto& c : cst) CKG_CUDA(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
      for (auto& e : gev) CKG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CKG_CUDA(cudaFuncSetAttribute(small_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kSmallSort * sizeof(unsigned long long))));
    }
    if (fexec[c0]) {
      CKG_CUDA(cudaGraphExecDestroy(fexec[c0]));
      fexec[c0] = nullptr;
    }
    cudaGraph_t g;
    CKG_CUDA(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hw;
    CKG_CUDA(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = hw;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t wn;
    CKG_CUDA(cudaGraphAddNode(&wn, g, nullptr, 0, &p));
    cudaGraph_t body = p.conditional.phGraph_out[0];
    uint32_t* const saved_perm = perm;
    uint32_t* const saved_skeys = skeys;
    CKG_CUDA(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    cudaGraphConditionalHandle hi;
    CKG_CUDA(cudaGraphConditionalHandleCreate(&hi, capture_graph_of(st), 0, cudaGraphCondAssignDefault));
    capture_graph_substep(st, cst[0], c0, hw, hi, cst[3], gev[0], gev[1]);
    cudaGraph_t second = add_conditional(st, hi, cudaGraphCondTypeIf);
    CKG_CUDA(cudaStreamBeginCaptureToGraph(cst[1], second, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    capture_graph_substep(cst[1], cst[2], c0 ^ 1, hw, hw, cst[4], gev[2], gev[3]);
    cudaGraph_t done;
    CKG_CUDA(cudaStreamEndCapture(cst[1], &done));
    CKG_CUDA(cudaStreamEndCapture(st, &done));
    CKG_CUDA(cudaGraphInstantiate(&fexec[c0], g, 0));
    CKG_CUDA(cudaGraphDestroy(g));
    perm = saved_perm;
    skeys = saved_skeys;
    fkey[c0] = graph_key();
  }

  // The graph needs: the stored-order keys (incremental sort), a valid stress
  // cache, a pool that cannot overflow (sized for the whole directory) and a
  // single domain.
  bool graph_ready() const {
    return !fused && !det && !slab && n > 0 && ko_valid && stress_valid && pool_cap >= nd;
  }

  // Host-side bookkeeping of one completed host-loop substep (gather_all + the
  // loop body of advance_frame).  Returns true when the frame continues.
  bool host_substep(FrameState& fs, ckg_frame_out* out, int& rc) {
    const T rem = T(fs.frame_end) - T(fs.time);
    const T dt = host_cfl_dt(fs, rem);
    ckg_step_out so;
    rc = step(double(dt), CKG_PHASE_G2P, 1, &so);
    out->kernel_launches += so.kernel_launches;
    out->active_blocks = so.active_blocks;
    if (rc != CKG_OK) {
      out->error_code = so.error_code;
      out->error_axis = so.error_axis;
      out->error_phase = so.error_phase;
      out->error_particle = so.error_particle;
      return false;
    }
    fs.vmax = so.vmax;
    for (int m = 0; m < kMaxMaterials; ++m) fs.min_j[m] = so.min_j[m];
    fs.time = double(T(fs.time) + dt);
    fs.dt = double(dt);
    fs.substeps += 1;
    if (fs.substeps > fs.max_substeps) {
      fs.status = 3;
      return false;
    }
    const T r2 = T(fs.frame_end) - T(fs.time);
    if (r2 <= T(fs.frame_dt) * T(1e-9)) {
      fs.time = fs.frame_end;
      fs.status = 1;
      return false;
    }
    return true;
  }

  int advance_frame(const ckg_frame_in* in, ckg_frame_out* out) override {
    CKG_CUDA(cudaSetDevice(device));
    std::memset(out, 0, sizeof(*out));
    FrameState fs{};
    const T frame_dt = T(in->frame_dt);
    fs.frame_dt = double(frame_dt);
    fs.frame_end = double(frame_dt * T(double(in->frame_index + 1)));
    fs.time = double(T(in->time));
    fs.cfl = in->cfl;
    fs.max_dt = in->max_dt;
    fs.vmax = in->vmax;
    for (int m = 0; m < kMaxMaterials; ++m) fs.min_j[m] = in->min_j[m];
    fs.max_substeps = uint32_t(std::min<uint64_t>(in->max_substeps, 0xfffffff0u));
    fs.status = 0;
    int rc = CKG_OK;
    const uint64_t steps0 = step_count;
    auto finish = [&](int code) {
      out->substeps = fs.substeps;
      out->time = fs.time;
      out->last_dt = fs.dt;
      out->vmax = fs.vmax;
      for (int m = 0; m < kMaxMaterials; ++m) out->min_j[m] = fs.min_j[m];
      for (int k = 0; k < 3; ++k) out->sort_paths[k] = fs.sort_paths[k];
      if (fs.status == 3) {
        last_error = "substep limit exceeded within one frame at t = " + std::to_string(double(T(fs.time)));
        out->error_code = CKG_NUM_SUBSTEP_LIMIT;
        code = CKG_ERR_NUMERICAL;
      }
      out->status = code;
      return code;
    };
    {
      const T rem = T(fs.frame_end) - T(fs.time);
      if (rem <= frame_dt * T(1e-9)) {
        fs.time = fs.frame_end;
        fs.status = 1;
        return finish(CKG_OK);
      }
    }
    // substeps the graph cannot run yet go through the host loop
    while (!graph_ready()) {
      if (!host_substep(fs, out, rc)) return finish(rc);
    }
    out->graph = 1;
    const int c0 = cur;
    if (!fexec[c0] || !(fkey[c0] == graph_key())) build_frame_graph(c0);
    fs.parity = uint32_t(cur);
    *hframe = fs;
    CKG_CUDA(cudaMemcpyAsync(dframe, hframe, sizeof(FrameState), cudaMemcpyHostToDevice, st));
    CKG_CUDA(cudaEventRecord(tev[14], st));
    CKG_CUDA(cudaGraphLaunch(fexec[c0], st));
    CKG_CUDA(cudaEventRecord(tev[15], st));
    CKG_CUDA(cudaMemcpyAsync(hframe, dframe, sizeof(FrameState), cudaMemcpyDeviceToHost, st));
    CKG_CUDA(cudaMemcpyAsync(hstat, dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
    CKG_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    cudaEventElapsedTime(&ms, tev[14], tev[15]);
    out->device_ms = ms;
    const uint32_t graph_steps = hframe->substeps - fs.substeps;
    fs = *hframe;
    cur = int(fs.parity);
    step_count = steps0 + fs.substeps;
    out->kernel_launches += uint64_t(graph_steps + (fs.status == 2 ? 1 : 0)) * graph_kernels;
    out->active_blocks = hstat->n_active;
    grid_valid = true;
    last_active = hstat->n_active;
    perm = perm_buf;
    skeys = ko;
    if (fs.status == 2) {
      ko_valid = false;  // the failing substep re-sorted; the stored order did not move
      ckg_step_out so;
      std::memset(&so, 0, sizeof so);
      if (hstat->overflow) {
        last_error = "grid block pool capacity exceeded";
        return finish(CKG_ERR_DEVICE);
      }
      const int code = decode_status(&so, CKG_PHASE_G2P);
      out->error_code = so.error_code;
      out->error_axis = so.error_axis;
      out->error_phase = so.error_phase;
      out->error_particle = so.error_particle;
      return finish(code);
    }
    return finish(CKG_OK);
  }

  // ---------------------------------------------------------------- checkpoint / snapshot
  uint64_t record_bytes(int kind) const override {
    return kind == CKG_RECORDS_CHECKPOINT ? uint64_t(checkpoint_words<T>()) * 4 : uint64_t(kSnapshotWords) * 4;
  }

  int pack_records(int kind, void* host, uint64_t bytes, int async) override {
    if (kind != CKG_RECORDS_CHECKPOINT && kind != CKG_RECORDS_SNAPSHOT) {
      last_error = "records: unknown kind";
      return CKG_ERR_CONFIG;
    }
    const uint64_t need = n * record_bytes(kind);
    if (bytes < need) {
      last_error = "records: host buffer too small";
      return CKG_ERR_CONFIG;
    }
    if (n == 0) return CKG_OK;
    CKG_CUDA(cudaSetDevice(device));
    if (!iost) {
      CKG_CUDA(cudaStreamCreateWithFlags(&iost, cudaStreamNonBlocking));
      CKG_CUDA(cudaEventCreateWithFlags(&io_packed, cudaEventDisableTiming));
      CKG_CUDA(cudaEventCreateWithFlags(&io_done, cudaEventDisableTiming));
    }
    if (io_pending) CKG_CUDA(cudaStreamWaitEvent(st, io_done, 0));  // the previous copy still reads iobuf
    const uint64_t words = need / 4;
    if (words > iobuf_words) {
      CKG_CUDA(cudaStreamSynchronize(st));
      dfree(iobuf);
      iobuf = dalloc<uint32_t>(words);
      iobuf_words = words;
    }
    uint32_t fluid = 0;
    for (int m = 0; m < cfg.n_materials && m < 32; ++m)
      if (cfg.materials[m].model == CKG_MODEL_J_FLUID) fluid |= 1u << m;
    pack_records_kernel<T><<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(state(cur), kind, fluid, iobuf);
    CKG_CUDA(cudaGetLastError());
    CKG_CUDA(cudaEventRecord(io_packed, st));
    CKG_CUDA(cudaStreamWaitEvent(iost, io_packed, 0));
    CKG_CUDA(cudaMemcpyAsync(host, iobuf, need, cudaMemcpyDeviceToHost, iost));
    CKG_CUDA(cudaEventRecord(io_done, iost));
    io_pending = true;
    if (!async) return records_wait();
    return CKG_OK;
  }

  int records_wait() override {
    if (io_pending) {
      CKG_CUDA(cudaEventSynchronize(io_done));
      io_pending = false;
    }
    return CKG_OK;
  }

  int debug_sort(uint32_t* hkeys, uint32_t* horder, uint64_t count) override {
    if (count != n) return CKG_ERR_CONFIG;
    if (n == 0) return CKG_OK;
    CKG_CUDA(cudaSetDevice(device));
    status_reset_kernel<<<1, 32, 0, st>>>(dstat, 1);
    enqueue_sort();
    CKG_CUDA(cudaMemcpyAsync(hkeys, skeys, n * 4, cudaMemcpyDeviceToHost, st));
    CKG_CUDA(cudaMemcpyAsync(horder, perm, n * 4, cudaMemcpyDeviceToHost, st));
    CKG_CUDA(cudaMemsetAsync(core, 0, nd * sizeof(uint32_t), st));
    CKG_CUDA(cudaStreamSynchronize(st));
    ko_valid = false;  // the stored order was not permuted
    return CKG_OK;
  }

  int debug_bases(int32_t* hb, uint64_t count) override {
    if (count != n) return CKG_ERR_CONFIG;
    if (n == 0) return CKG_OK;
    CKG_CUDA(cudaSetDevice(device));
    int32_t* d = dalloc<int32_t>(n * 6);
    const StepConst<T> c = make_const(0.0);
    bases_kernel<T><<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(state(cur), c.dx, c.inv_dx, c.pow2, d);
    CKG_CUDA(cudaMemcpyAsync(hb, d, n * 6 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CKG_CUDA(cudaStreamSynchronize(st));
    cudaFree(d);
    return CKG_OK;
  }

  uint64_t active_blocks() override { return grid_valid ? std::min<uint64_t>(last_active, pool_cap) : 0; }

  int grid_download(int32_t* coords, double* nodes, uint64_t nb) override {
    CKG_CUDA(cudaSetDevice(device));
    nb = std::min<uint64_t>(nb, active_blocks());
    if (nb == 0) return CKG_OK;
    int32_t* dc = coords ? dalloc<int32_t>(nb * 3) : nullptr;
    double* dn = nodes ? dalloc<double>(nb * 128 * 4) : nullptr;
    grid_export_kernel<T><<<grid_for(nb * 128, 256), 256, 0, st>>>(fused ? facade_pool : pool, active, nb, D, dc,
                                                                   dn, fused ? 1 : 0);
    CKG_CUDA(cudaGetLastError());
    if (dc) CKG_CUDA(cudaMemcpyAsync(coords, dc, nb * 3 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    if (dn) CKG_CUDA(cudaMemcpyAsync(nodes, dn, nb * 512 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CKG_CUDA(cudaStreamSynchronize(st));
    if (dc) cudaFree(dc);
    if (dn) cudaFree(dn);
    return CKG_OK;
  }

  int grid_totals(double* mass, double* mom) override {
    uint64_t nb = active_blocks();
    std::vector<double> nodes(std::max<uint64_t>(nb, 1) * 512);
    for (int g = 0; g < 2; ++g) {
      mass[g] = 0;
      for (int a = 0; a < 3; ++a) mom[g * 3 + a] = 0;
    }
    if (nb == 0) return CKG_OK;
    int rc = grid_download(nullptr, nodes.data(), nb);
    if (rc) return rc;
    // Same summation order as BlockSparseGrid::total_mass (grid.hpp:199-213)
    // over blocks in directory order.
    for (uint64_t b = 0; b < nb; ++b)
      for (int g = 0; g < 2; ++g)
        for (int l = 0; l < 64; ++l) {
          const double* o = &nodes[(b * 128 + g * 64 + l) * 4];
          mass[g] += o[0];
          for (int a = 0; a < 3; ++a) mom[g * 3 + a] += o[1 + a];
        }
    return CKG_OK;
  }

  // ---------------------------------------------------------------- slabs
  // Staged substep for the x-slab decomposition; the host moves the
  // exchange buffers between stages (paper_2412_10399_b200/slab.py).
  bool force_full_relayout = false;  // CKMPM_SLAB_FULL_RELAYOUT=1: always take the full migration path (tests)

  int slab_set(int rank, int world, int lo, int hi) override {
    if (lo < 0 || hi > D || lo >= hi || rank < 0 || rank >= world) return CKG_ERR_CONFIG;
    disable_fused();
    slab = true;
    const char* env = std::getenv("CKMPM_SLAB_FULL_RELAYOUT");
    force_full_relayout = env && env[0] == '1';
    srank = rank;
    sworld = world;
    bx_lo = lo;
    bx_hi = hi;
    CKG_CUDA(cudaSetDevice(device));
    dfree(plane_start);
    plane_start = dalloc<uint32_t>(uint64_t(D) + 1);
    if (det) set_det_cap(std::min<uint32_t>(pool_cap, 1u << 18));  // slots are global: every rank's blocks
    return CKG_OK;
  }

  // Rebalancing: the new slab [lo, hi) takes effect at this substep's
  // migration (its P2G, grid update and halos still use the old bounds);
  // slab_finish commits it.  Particles of planes that change hands travel
  // with the substep's migrants (full relayout path).
  int slab_rebound(int lo, int hi) override {
    if (!slab || lo < 0 || hi > D || lo >= hi) return CKG_ERR_CONFIG;
    pend_lo = lo;
    pend_hi = hi;
    return CKG_OK;
  }

  // Particles of the current state per key plane bx (D counters).
  int slab_plane_counts(uint64_t* counts) override {
    CKG_CUDA(cudaSetDevice(device));
    unsigned long long* d = dalloc<unsigned long long>(uint64_t(D));
    CKG_CUDA(cudaMemsetAsync(d, 0, uint64_t(D) * sizeof(unsigned long long), st));
    if (n) plane_count_kernel<T><<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(state(cur), T(cfg.inv_dx), D, d);
    CKG_CUDA(cudaMemcpyAsync(counts, d, uint64_t(D) * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CKG_CUDA(cudaStreamSynchronize(st));
    cudaFree(d);
    return CKG_OK;
  }

  int plane_bx(int sel) const {
    return sel == 0 ? bx_lo - 1 : sel == 1 ? bx_lo : sel == 2 ? bx_hi - 1 : bx_hi;
  }

  int slab_bin(double dt, void* core_out) override {
    if (!slab) return CKG_ERR_CONFIG;
    CKG_CUDA(cudaSetDevice(device));
    launches = 0;
    slab_dt = dt;
    status_reset_kernel<<<1, 32, 0, st>>>(dstat, 1);
    CKG_CUDA(cudaEventRecord(ev[0], st));
    enqueue_sort();
    CKG_CUDA(cudaMemcpyAsync(core_out, core, nd * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    CKG_CUDA(cudaStreamSynchronize(st));
    return CKG_OK;
  }

  template <int S>
  void enqueue_p2g_range(const StepConst<T>& c, int a, int b) {
    slab_item_range_kernel<<<1, 1, 0, st>>>(plane_start, a, b, dstat);
    enqueue_p2g<S>(c, 0);
  }
  void enqueue_p2g_range_any(const StepConst<T>& c, int a, int b) {
    if (cfg.scheme == CKG_SCHEME_PIC) enqueue_p2g_range<kSchemePic>(c, a, b);
    else if (cfg.scheme == CKG_SCHEME_APIC) enqueue_p2g_range<kSchemeApic>(c, a, b);
    else enqueue_p2g_range<kSchemeMls>(c, a, b);
  }

  // part 0: activation + the whole P2G; 1: activation + the P2G of the two
  // boundary planes (bx_lo, bx_hi - 1: the only ones whose tiles reach the
  // ghost planes); 2: the interior planes' P2G (the halo exchange of part 1's
  // ghost planes can run meanwhile).  Parts 0 and 1 return the block counts
  // of planes ghostL, ownL, ownR, ghostR.
  int slab_p2g(const void* core_in, uint64_t* plane_blocks, int part) override {
    CKG_CUDA(cudaSetDevice(device));
    const StepConst<T> c = make_const(slab_dt);
    if (part == 2) {
      if (bx_hi - bx_lo > 2) enqueue_p2g_range_any(c, bx_lo + 1, bx_hi - 1);
      slab_item_range_kernel<<<1, 1, 0, st>>>(plane_start, bx_lo, bx_hi, dstat);  // G2P's range
      CKG_CUDA(cudaEventRecord(ev[4], st));
      launches += 3;
      return CKG_OK;
    }
    CKG_CUDA(cudaMemcpyAsync(core, core_in, nd * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    CKG_CUDA(cudaEventRecord(ev[1], st));
    enqueue_activate(0);
    CKG_CUDA(cudaEventRecord(ev[2], st));
    clear_kernel<T><<<148 * 8, 256, 0, st>>>(pool, dstat, pool_cap);
    CKG_CUDA(cudaEventRecord(ev[3], st));
    if (!stress_valid) {
      stress_kernel<T><<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(state(cur), perm, c, dstat, 0);
      stress_valid = true;
    }
    if (part == 1) {
      enqueue_p2g_range_any(c, bx_lo, bx_lo + 1);
      if (bx_hi - 1 > bx_lo) enqueue_p2g_range_any(c, bx_hi - 1, bx_hi);
      launches += 4;
    } else {
      if (cfg.scheme == CKG_SCHEME_PIC) enqueue_p2g<kSchemePic>(c, 0);
      else if (cfg.scheme == CKG_SCHEME_APIC) enqueue_p2g<kSchemeApic>(c, 0);
      else enqueue_p2g<kSchemeMls>(c, 0);
      CKG_CUDA(cudaEventRecord(ev[4], st));
    }
    launches += 12;
    std::vector<uint32_t> ps(uint64_t(D) + 1);
    CKG_CUDA(cudaMemcpyAsync(ps.data(), plane_start, ps.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CKG_CUDA(cudaStreamSynchronize(st));
    for (int sel = 0; sel < 4; ++sel) {
      const int bx = plane_bx(sel);
      plane_blocks[sel] = (bx < 0 || bx >= D) ? 0 : uint64_t(ps[bx + 1] - ps[bx]);
    }
    return CKG_OK;
  }

  // op 0: pack plane -> buf, 1: add buf into plane, 2: copy buf into plane;
  // deterministic mode: 3 pack the plane's P2G tiles, 4 copy buf into them
  int slab_halo(int op, int sel, void* buf) override {
    const int bx = plane_bx(sel);
    if (bx < 0 || bx >= D) return CKG_OK;
    CKG_CUDA(cudaSetDevice(device));
    if (op == 3 || op == 4) {
      if (!det) return CKG_ERR_CONFIG;
      tile_halo_kernel<T><<<148 * 4, 256, 0, st>>>(dtile, dcap, plane_start, bx, op, static_cast<T*>(buf),
                                                   &dstat->overflow);
      launches += 1;
      return CKG_OK;
    }
    // stream-ordered: an exchange enqueued on this stream (ckg_stream) sees
    // the packed buffer; a host or another stream synchronises first
    halo_kernel<T><<<148 * 4, 256, 0, st>>>(pool, plane_start, bx, op, static_cast<T*>(buf));
    launches += 1;
    return CKG_OK;
  }

  int slab_grid() override {
    CKG_CUDA(cudaSetDevice(device));
    const StepConst<T> c = make_const(slab_dt);
    if (det) enqueue_det_gather();  // own planes, from local and received tiles
    grid_update_kernel<T><<<148 * 8, 256, 0, st>>>(pool, active, dstat, pool_cap, c, dbcs);
    CKG_CUDA(cudaEventRecord(ev[5], st));
    launches += 1;
    return CKG_OK;
  }

  int slab_g2p(uint64_t* counts) override {
    CKG_CUDA(cudaSetDevice(device));
    const StepConst<T> c = make_const(slab_dt);
    wb[cur ^ 1] = wb[cur];  // G2P writes the new state at the same window
    if (cfg.scheme == CKG_SCHEME_PIC) enqueue_g2p<kSchemePic>(c, 0);
    else if (cfg.scheme == CKG_SCHEME_APIC) enqueue_g2p<kSchemeApic>(c, 0);
    else enqueue_g2p<kSchemeMls>(c, 0);
    CKG_CUDA(cudaEventRecord(ev[6], st));
    PState<T> nx = state(cur ^ 1);
    const bool rebound = pend_lo >= 0;
    classify_kernel<T><<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(nx, T(cfg.inv_dx), D, rebound ? pend_lo : bx_lo,
                                                                   rebound ? pend_hi : bx_hi, fl_stay, fl_left,
                                                                   fl_right);
    launches += 2;
    // crossers can only come from the first and last owned plane: find the
    // sorted regions of those planes and check the middle holds none
    if (!dreg) dreg = dalloc<unsigned long long>(3);
    CKG_CUDA(cudaMemsetAsync(dreg, 0, 3 * sizeof(unsigned long long), st));
    const uint64_t DD = uint64_t(D) * D;
    slab_regions_kernel<<<1, 1, 0, st>>>(skeys, n, uint32_t((bx_lo + 1) * DD), uint32_t((bx_hi - 1) * DD), dreg);
    unsigned long long hreg[3] = {0, 0, 0};
    CKG_CUDA(cudaMemcpyAsync(hreg, dreg, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CKG_CUDA(cudaStreamSynchronize(st));
    reg_pl = hreg[0];
    reg_pr = hreg[1];
    mig_region = !force_full_relayout && !rebound && bx_hi - bx_lo >= 2 && reg_pl <= reg_pr;
    if (mig_region) {
      // no crosser in the middle, none leaving the "wrong" side of a region
      if (reg_pr > reg_pl)
        count_far_kernel<<<grid_for(reg_pr - reg_pl, 256, 148 * 8), 256, 0, st>>>(fl_left, fl_right, reg_pl, reg_pr,
                                                                                dreg + 2);
      if (reg_pl)
        count_far_kernel<<<grid_for(reg_pl, 256, 148 * 8), 256, 0, st>>>(fl_right, fl_right, 0, reg_pl, dreg + 2);
      if (n > reg_pr)
        count_far_kernel<<<grid_for(n - reg_pr, 256, 148 * 8), 256, 0, st>>>(fl_left, fl_left, reg_pr, n, dreg + 2);
      // region-local scans (left: [0, PL), right: [PR, n))
      const uint64_t nr = n - reg_pr;
      if (reg_pl) {
        exclusive_scan(fl_left, pos_left, reg_pl, scan_partials_n, st);
        exclusive_scan(fl_stay, pos_stay, reg_pl, scan_partials_n, st);
      }
      if (nr) {
        exclusive_scan(fl_right + reg_pr, pos_right, nr, scan_partials_n, st);
        exclusive_scan(fl_stay + reg_pr, pos_stay + reg_pl, nr, scan_partials_n, st);
      }
      launches += 13;
      uint32_t tail[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (reg_pl) {
        CKG_CUDA(cudaMemcpyAsync(&tail[0], pos_left + reg_pl - 1, 4, cudaMemcpyDeviceToHost, st));
        CKG_CUDA(cudaMemcpyAsync(&tail[1], fl_left + reg_pl - 1, 4, cudaMemcpyDeviceToHost, st));
      }
      if (nr) {
        CKG_CUDA(cudaMemcpyAsync(&tail[2], pos_right + nr - 1, 4, cudaMemcpyDeviceToHost, st));
        CKG_CUDA(cudaMemcpyAsync(&tail[3], fl_right + n - 1, 4, cudaMemcpyDeviceToHost, st));
      }
      CKG_CUDA(cudaMemcpyAsync(&hreg[2], dreg + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
      CKG_CUDA(cudaStreamSynchronize(st));
      if (hreg[2] == 0) {
        mig_left = uint64_t(tail[0]) + tail[1];
        mig_right = uint64_t(tail[2]) + tail[3];
        stay_l = reg_pl - mig_left;
        stay_r = nr - mig_right;
        n_stay = n - mig_left - mig_right;
        counts[0] = mig_left;
        counts[1] = mig_right;
        return CKG_OK;
      }
      mig_region = false;  // a crosser away from the boundary planes (dt beyond CFL): full path
    }
    exclusive_scan(fl_stay, pos_stay, n, scan_partials_n, st);
    exclusive_scan(fl_left, pos_left, n, scan_partials_n, st);
    exclusive_scan(fl_right, pos_right, n, scan_partials_n, st);
    launches += 9;
    uint32_t tail[6] = {0, 0, 0, 0, 0, 0};
    if (n) {
      CKG_CUDA(cudaMemcpyAsync(&tail[0], pos_stay + n - 1, 4, cudaMemcpyDeviceToHost, st));
      CKG_CUDA(cudaMemcpyAsync(&tail[1], fl_stay + n - 1, 4, cudaMemcpyDeviceToHost, st));
      CKG_CUDA(cudaMemcpyAsync(&tail[2], pos_left + n - 1, 4, cudaMemcpyDeviceToHost, st));
      CKG_CUDA(cudaMemcpyAsync(&tail[3], fl_left + n - 1, 4, cudaMemcpyDeviceToHost, st));
      CKG_CUDA(cudaMemcpyAsync(&tail[4], pos_right + n - 1, 4, cudaMemcpyDeviceToHost, st));
      CKG_CUDA(cudaMemcpyAsync(&tail[5], fl_right + n - 1, 4, cudaMemcpyDeviceToHost, st));
    }
    CKG_CUDA(cudaStreamSynchronize(st));
    n_stay = uint64_t(tail[0]) + tail[1];
    mig_left = uint64_t(tail[2]) + tail[3];
    mig_right = uint64_t(tail[4]) + tail[5];
    counts[0] = mig_left;
    counts[1] = mig_right;
    return CKG_OK;
  }

  int slab_pack(uint64_t nl_in, void* left, void* right) override {
    CKG_CUDA(cudaSetDevice(device));
    PState<T> nx = state(cur ^ 1);
    if (mig_region) {
      // window start after the exchange: wb + out_left - in_left must stay in
      // the buffer (else relayout through the full path below)
      const int64_t base = int64_t(wb[cur ^ 1]) + int64_t(mig_left) - int64_t(nl_in);
      if (base >= 0) {
        PState<T> tmp = state_at(cur, wb[cur ^ 1], n);  // the old state buffer, same window: scratch
        if (reg_pl)
          region_out_kernel<T><<<grid_for(reg_pl, 256, 1 << 30), 256, 0, st>>>(
              nx, skeys, 0, reg_pl, fl_left, pos_left, fl_right, pos_right, static_cast<T*>(left),
              static_cast<T*>(right), tmp);
        if (n > reg_pr)
          region_out_kernel<T><<<grid_for(n - reg_pr, 256, 1 << 30), 256, 0, st>>>(
              nx, skeys, reg_pr, n, fl_left, pos_left, fl_right, pos_right, static_cast<T*>(left),
              static_cast<T*>(right), tmp);
        launches += 2;
        CKG_CUDA(cudaStreamSynchronize(st));
        return CKG_OK;
      }
      mig_region = false;
      // the region scans are not the full ones the relayout needs
      exclusive_scan(fl_stay, pos_stay, n, scan_partials_n, st);
      exclusive_scan(fl_left, pos_left, n, scan_partials_n, st);
      exclusive_scan(fl_right, pos_right, n, scan_partials_n, st);
      launches += 9;
    }
    // full relayout into the other buffer, re-centred: survivors at
    // [nl_in, nl_in + n_stay) with their sorted keys of this substep (the
    // next substep's ko); migrants -> records
    const uint64_t total_max = nl_in + n_stay + std::max<uint64_t>(n, 1u << 20);
    if (nl_in + n_stay > cap) {
      last_error = "slab: particle capacity of this rank exceeded";
      return CKG_ERR_DEVICE;
    }
    wb[cur] = cap > total_max ? (cap - total_max) / 2 : 0;
    PState<T> dst = state(cur);
    migrate_out_kernel<T><<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(
        nx, skeys, fl_stay, pos_stay, fl_left, pos_left, fl_right, pos_right, dst, skeys_tmp, nl_in,
        static_cast<T*>(left), static_cast<T*>(right));
    launches += 1;
    CKG_CUDA(cudaStreamSynchronize(st));
    return CKG_OK;
  }

  int slab_finish(const void* left, uint64_t nl, const void* right, uint64_t nr, ckg_step_out* out) override {
    CKG_CUDA(cudaSetDevice(device));
    const uint64_t total = nl + n_stay + nr;
    const bool region = mig_region;
    if (mig_region) {
      const int nb = cur ^ 1;
      const uint64_t base = wb[nb] + mig_left - nl;
      if (base + total > cap) {
        last_error = "slab: particle capacity of this rank exceeded";
        return CKG_ERR_DEVICE;
      }
      // region survivors into place (old window coordinates), then the
      // next substep's keys, then the incoming migrants (new window)
      PState<T> tmp = state_at(cur, wb[nb], n);
      PState<T> old_win = state_at(nb, wb[nb], n);
      if (reg_pl)
        region_in_kernel<T><<<grid_for(reg_pl, 256, 1 << 30), 256, 0, st>>>(tmp, 0, reg_pl, fl_stay, pos_stay, old_win,
                                                                            int64_t(mig_left));
      if (n > reg_pr)
        region_in_kernel<T><<<grid_for(n - reg_pr, 256, 1 << 30), 256, 0, st>>>(
            tmp, reg_pr, n, fl_stay, pos_stay + reg_pl, old_win, int64_t(reg_pr));
      region_keys_kernel<<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(
          skeys, n, reg_pl, reg_pr, int64_t(nl) - int64_t(mig_left), fl_stay, pos_stay, pos_stay + reg_pl, nl,
          stay_l, skeys_tmp);
      PState<T> dst = state_at(nb, base, total);
      if (nl)
        migrate_in_kernel<T><<<grid_for(nl, 256, 1 << 30), 256, 0, st>>>(static_cast<const T*>(left), nl, dst,
                                                                         skeys_tmp, 0);
      if (nr)
        migrate_in_kernel<T><<<grid_for(nr, 256, 1 << 30), 256, 0, st>>>(static_cast<const T*>(right), nr, dst,
                                                                         skeys_tmp, total - nr);
      launches += 5;
      wb[nb] = base;
      cur = nb;
    } else {
      if (wb[cur] + total > cap) {
        last_error = "slab: particle capacity of this rank exceeded";
        return CKG_ERR_DEVICE;
      }
      PState<T> dst = state(cur);
      dst.n = total;
      if (nl)
        migrate_in_kernel<T><<<grid_for(nl, 256, 1 << 30), 256, 0, st>>>(static_cast<const T*>(left), nl, dst,
                                                                         skeys_tmp, 0);
      if (nr)
        migrate_in_kernel<T><<<grid_for(nr, 256, 1 << 30), 256, 0, st>>>(static_cast<const T*>(right), nr, dst,
                                                                         skeys_tmp, nl + n_stay);
      launches += 2;
    }
    std::swap(ko, skeys_tmp);
    ko_valid = true;  // [left keys][survivor keys][right keys] is non-decreasing
    n = total;
    CKG_CUDA(cudaMemcpyAsync(hstat, dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
    CKG_CUDA(cudaStreamSynchronize(st));
    ckg_step_out local;
    if (!out) out = &local;
    fill_out(out, true, CKG_PHASE_G2P);
    out->kernel_launches = launches;
    out->sort_changed = last_changed;
    out->sort_kind = last_sort_kind;
    out->slab_migration = region ? 1 : 2;
    grid_valid = true;
    last_active = hstat->n_active;
    if (pend_lo >= 0) {  // rebalanced slab committed
      bx_lo = pend_lo;
      bx_hi = pend_hi;
      pend_lo = pend_hi = -1;
    }
    if (hstat->overflow) {
      last_error = (hstat->overflow & 8u)
                       ? "deterministic x-slab mode: out-of-tile particles (needs a power-of-two cell size)"
                       : "grid block pool / deterministic tile buffer capacity exceeded";
      out->status = CKG_ERR_DEVICE;
      return CKG_ERR_DEVICE;
    }
    int rc = decode_status(out, CKG_PHASE_G2P);
    if (rc == CKG_OK) step_count += 1;
    out->status = rc;
    return rc;
  }

  int timer_mark(int slot) override {
    if (slot < 0 || slot >= 16) return CKG_ERR_CONFIG;
    CKG_CUDA(cudaEventRecord(tev[slot], st));
    return CKG_OK;
  }

  int timer_elapsed(int a, int b, double* ms) override {
    if (a < 0 || a >= 16 || b < 0 || b >= 16 || !ms) return CKG_ERR_CONFIG;
    CKG_CUDA(cudaEventSynchronize(tev[b]));
    float f = 0;
    CKG_CUDA(cudaEventElapsedTime(&f, tev[a], tev[b]));
    *ms = f;
    return CKG_OK;
  }

  int diagnostics(ckg_diagnostics* out) override {
    std::memset(out, 0, sizeof(*out));
    if (n == 0) return CKG_OK;
    CKG_CUDA(cudaSetDevice(device));
    CKG_CUDA(cudaMemsetAsync(dacc, 0, 12 * sizeof(double), st));
    diagnostics_kernel<T><<<grid_for(n, 256, 148 * 4), 256, 0, st>>>(
        state(cur), dacc, reinterpret_cast<unsigned long long*>(dacc + 10));
    double h[12];
    CKG_CUDA(cudaMemcpyAsync(h, dacc, sizeof h, cudaMemcpyDeviceToHost, st));
    CKG_CUDA(cudaStreamSynchronize(st));
    for (int a = 0; a < 3; ++a) {
      out->momentum[a] = h[a];
      out->angular[a] = h[3 + a];
      out->momentum_massfree[a] = h[6 + a];
    }
    out->kinetic_energy = h[9];
    double vm2;
    std::memcpy(&vm2, &h[10], sizeof vm2);
    out->vmax = std::sqrt(vm2);
    return CKG_OK;
  }
};

}  // namespace ckg

struct ckg_ctx {
  std::unique_ptr<ckg::CtxBase> impl;
  std::string err;
};

namespace {

int32_t guard(ckg_ctx* ctx, const char* where, const std::function<int32_t()>& f) {
  try {
    return f();
  } catch (const ckg::CudaError& e) {
    if (ctx) ctx->err = std::string(where) + ": CUDA error " + cudaGetErrorString(e.e) + " in " + e.what;
    std::fprintf(stderr, "[ckmpm_b200] %s: CUDA error %s in %s\n", where, cudaGetErrorString(e.e), e.what);
    return CKG_ERR_DEVICE;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->err = std::string(where) + ": host allocation failed";
    return CKG_ERR_DEVICE;
  }
}

std::string validate(const ckg_config* c) {
  if (!c) return "config: null";
  if (c->abi_version != CKG_ABI_VERSION) return "config: ABI version mismatch";
  if (c->precision != 8 && c->precision != 4) return "precision: must be 4 or 8";
  if (c->resolution < 8) return "resolution: must be at least 8";
  if (!(c->extent > 0)) return "extent: must be positive";
  if (!(c->dx > 0) || !(c->inv_dx > 0)) return "grid dx must be positive";
  if (c->scheme < 0 || c->scheme > 2) return "scheme: expected 'pic', 'apic' or 'mls'";
  if (c->n_materials < 1) return "materials: at least one required";
  if (c->n_materials > CKG_MAX_MATERIALS) return "materials: too many for the device table";
  if (c->n_boundaries < 0 || c->n_boundaries > CKG_MAX_BOUNDARIES) return "boundaries: too many";
  for (int m = 0; m < c->n_materials; ++m) {
    int model = c->materials[m].model;
    if (model != CKG_MODEL_FIXED_COROTATED && model != CKG_MODEL_J_FLUID && model != CKG_MODEL_DRUCKER_PRAGER)
      return "material: reserved tag and not implemented";
  }
  if (c->flags & ~(CKG_FLAG_QUADRATIC | CKG_FLAG_FUSED)) return "config: unknown flags";
  if ((c->flags & CKG_FLAG_QUADRATIC) && c->scheme == CKG_SCHEME_MLS)
    return "scheme: mls requires the compact kernel";  // scene.hpp:193-194
  long long D = c->resolution / 4 + 2;
  if (D * D * D >= (1ll << 31)) return "resolution: too large for the block directory";
  return {};
}

}  // namespace

extern "C" {

int32_t ckg_abi_version(void) { return CKG_ABI_VERSION; }

const char* ckg_build_info(void) {
  return "ckmpm_b200 abi 1; sm_100a";
}

const char* ckg_status_string(int32_t s) {
  switch (s) {
    case CKG_OK: return "ok";
    case CKG_ERR_CONFIG: return "ConfigError";
    case CKG_ERR_NUMERICAL: return "NumericalError";
    case CKG_ERR_IO: return "IoError";
    case CKG_ERR_DEVICE: return "DeviceError";
    default: return "unknown";
  }
}

int32_t ckg_create(const ckg_config* cfg, ckg_ctx** out) {
  if (!out) return CKG_ERR_CONFIG;
  *out = nullptr;
  std::string v = validate(cfg);
  if (!v.empty()) {
    std::fprintf(stderr, "[ckmpm_b200] ckg_create: %s\n", v.c_str());
    return CKG_ERR_CONFIG;
  }
  auto* ctx = new ckg_ctx();
  int32_t rc = guard(ctx, "ckg_create", [&]() -> int32_t {
    int ndev = 0;
    { cudaError_t e_ = cudaGetDeviceCount(&ndev); if (e_ != cudaSuccess) throw ckg::CudaError{e_, "cudaGetDeviceCount"}; }
    if (cfg->device < 0 || cfg->device >= ndev) throw ckg::CudaError{cudaErrorInvalidDevice, "device ordinal"};
    if (cfg->precision == 8)
      ctx->impl.reset(new ckg::Context<double>(*cfg));
    else
      ctx->impl.reset(new ckg::Context<float>(*cfg));
    return CKG_OK;
  });
  if (rc != CKG_OK) {
    delete ctx;
    return rc;
  }
  *out = ctx;
  return CKG_OK;
}

void ckg_destroy(ckg_ctx* ctx) { delete ctx; }

int32_t ckg_upload(ckg_ctx* ctx, const void* particles, uint64_t n) {
  if (!ctx || (!particles && n)) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_upload", [&] { return ctx->impl->upload(particles, n); });
}

int32_t ckg_download(ckg_ctx* ctx, void* particles, uint64_t n) {
  if (!ctx || (!particles && n)) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_download", [&] { return ctx->impl->download(particles, n); });
}

uint64_t ckg_particle_count(const ckg_ctx* ctx) { return ctx ? ctx->impl->count() : 0; }
int32_t ckg_fused(const ckg_ctx* ctx) { return ctx && ctx->impl->is_fused() ? 1 : 0; }
int32_t ckg_slab_tile_words(void) { return ckg::kDetVals; }
void* ckg_stream(ckg_ctx* ctx) { return ctx ? ctx->impl->stream() : nullptr; }

int32_t ckg_set_mass_epsilon(ckg_ctx* ctx, double eps) {
  if (!ctx) return CKG_ERR_CONFIG;
  ctx->impl->cfg.mass_eps = eps;
  return CKG_OK;
}

int32_t ckg_step(ckg_ctx* ctx, double dt, ckg_step_out* out) {
  if (!ctx) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_step", [&] { return ctx->impl->step(dt, CKG_PHASE_G2P, 1, out); });
}

int32_t ckg_step_many(ckg_ctx* ctx, double dt, int32_t count, ckg_step_out* out) {
  if (!ctx || count < 1 || count > 255) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_step_many", [&] { return ctx->impl->step(dt, CKG_PHASE_G2P, count, out); });
}

int32_t ckg_advance_frame(ckg_ctx* ctx, const ckg_frame_in* in, ckg_frame_out* out) {
  if (!ctx || !in || !out || !(in->frame_dt > 0)) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_advance_frame", [&] { return ctx->impl->advance_frame(in, out); });
}

uint64_t ckg_record_bytes(const ckg_ctx* ctx, int32_t kind) { return ctx ? ctx->impl->record_bytes(kind) : 0; }

int32_t ckg_pack_records(ckg_ctx* ctx, int32_t kind, void* host, uint64_t bytes, int32_t async) {
  if (!ctx || !host) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_pack_records", [&] { return ctx->impl->pack_records(kind, host, bytes, async); });
}

int32_t ckg_records_wait(ckg_ctx* ctx) {
  if (!ctx) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_records_wait", [&] { return ctx->impl->records_wait(); });
}

int32_t ckg_step_phases(ckg_ctx* ctx, double dt, int32_t stop_after, ckg_step_out* out) {
  if (!ctx || stop_after < CKG_PHASE_SORT || stop_after > CKG_PHASE_G2P) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_step_phases", [&] { return ctx->impl->step(dt, stop_after, 1, out); });
}

int32_t ckg_debug_sort(ckg_ctx* ctx, uint32_t* keys, uint32_t* order, uint64_t n) {
  if (!ctx || (n && (!keys || !order))) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_debug_sort", [&] { return ctx->impl->debug_sort(keys, order, n); });
}

int32_t ckg_debug_bases(ckg_ctx* ctx, int32_t* bases, uint64_t n) {
  if (!ctx || (n && !bases)) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_debug_bases", [&] { return ctx->impl->debug_bases(bases, n); });
}

uint64_t ckg_grid_active_block_count(ckg_ctx* ctx) { return ctx ? ctx->impl->active_blocks() : 0; }

int32_t ckg_grid_download(ckg_ctx* ctx, int32_t* coords, double* nodes, uint64_t nb) {
  if (!ctx) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_grid_download", [&] { return ctx->impl->grid_download(coords, nodes, nb); });
}

int32_t ckg_grid_totals(ckg_ctx* ctx, double mass[2], double momentum[6]) {
  if (!ctx || !mass || !momentum) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_grid_totals", [&] { return ctx->impl->grid_totals(mass, momentum); });
}

int32_t ckg_diagnostics_compute(ckg_ctx* ctx, ckg_diagnostics* out) {
  if (!ctx || !out) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_diagnostics_compute", [&] { return ctx->impl->diagnostics(out); });
}

int32_t ckg_slab_rebound(ckg_ctx* ctx, int32_t bx_lo, int32_t bx_hi) {
  if (!ctx) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_slab_rebound", [&] { return ctx->impl->slab_rebound(bx_lo, bx_hi); });
}
int32_t ckg_slab_plane_counts(ckg_ctx* ctx, uint64_t* counts) {
  if (!ctx || !counts) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_slab_plane_counts", [&] { return ctx->impl->slab_plane_counts(counts); });
}
int32_t ckg_slab_set(ckg_ctx* ctx, int32_t rank, int32_t world, int32_t bx_lo, int32_t bx_hi) {
  if (!ctx) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_slab_set", [&] { return ctx->impl->slab_set(rank, world, bx_lo, bx_hi); });
}
int32_t ckg_slab_bin(ckg_ctx* ctx, double dt, void* core_out) {
  if (!ctx || !core_out) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_slab_bin", [&] { return ctx->impl->slab_bin(dt, core_out); });
}
int32_t ckg_slab_p2g(ckg_ctx* ctx, const void* core_in, uint64_t plane_blocks[4]) {
  return guard(ctx, "ckg_slab_p2g", [&] { return ctx->impl->slab_p2g(core_in, plane_blocks, 0); });
}

int32_t ckg_slab_p2g_part(ckg_ctx* ctx, const void* core_in, uint64_t plane_blocks[4], int32_t part) {
  if (!ctx || part < 0 || part > 2) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_slab_p2g_part", [&] { return ctx->impl->slab_p2g(core_in, plane_blocks, part); });
}
int32_t ckg_slab_halo(ckg_ctx* ctx, int32_t op, int32_t plane, void* buf) {
  if (!ctx || op < 0 || op > 6 || plane < 0 || plane > 3) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_slab_halo", [&] { return ctx->impl->slab_halo(op, plane, buf); });
}
int32_t ckg_slab_grid(ckg_ctx* ctx) {
  if (!ctx) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_slab_grid", [&] { return ctx->impl->slab_grid(); });
}
int32_t ckg_slab_g2p(ckg_ctx* ctx, uint64_t counts[2]) {
  if (!ctx || !counts) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_slab_g2p", [&] { return ctx->impl->slab_g2p(counts); });
}
int32_t ckg_slab_pack(ckg_ctx* ctx, uint64_t nl_in, void* left, void* right) {
  if (!ctx) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_slab_pack", [&] { return ctx->impl->slab_pack(nl_in, left, right); });
}
int32_t ckg_slab_finish(ckg_ctx* ctx, const void* left, uint64_t nl, const void* right, uint64_t nr,
                        ckg_step_out* out) {
  if (!ctx) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_slab_finish", [&] { return ctx->impl->slab_finish(left, nl, right, nr, out); });
}
int32_t ckg_slab_record_words(void) { return ckg::kMigrantWords; }

int32_t ckg_timer_mark(ckg_ctx* ctx, int32_t slot) {
  if (!ctx) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_timer_mark", [&] { return ctx->impl->timer_mark(slot); });
}

int32_t ckg_timer_elapsed(ckg_ctx* ctx, int32_t a, int32_t b, double* ms) {
  if (!ctx) return CKG_ERR_CONFIG;
  return guard(ctx, "ckg_timer_elapsed", [&] { return ctx->impl->timer_elapsed(a, b, ms); });
}

int32_t ckg_last_error_message(ckg_ctx* ctx, char* buf, uint64_t cap) {
  if (!ctx || !buf || cap == 0) return CKG_ERR_CONFIG;
  const std::string& s = ctx->impl && !ctx->impl->last_error.empty() ? ctx->impl->last_error : ctx->err;
  std::snprintf(buf, cap, "%s", s.c_str());
  return CKG_OK;
}

}  // extern "C"
