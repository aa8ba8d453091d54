// capi.cpp -- the host runtime behind include/chemora.h: grid handles over a caller-owned
// workspace, stage sequencing of the RK4 step, the z-slab
// decomposition and its peer connectivity, and error reporting.
#include "../../include/chemora.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges for nsys timelines (no-ops without a tool)

#include "grid.hpp"
#include "kernels.hpp"

using namespace chemora;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return fail(CHEMORA_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));  \
  } while (0)

const double kBenchGauge[10] = {2.0, 1.0, 1.0, 0.0, 1.0, 0.75, 0.0, 1.0, 1.0, 1.0};
constexpr int kParams = 10;

struct PeerRecord {
  cudaIpcMemHandle_t handle;
  uint64_t offset;   // workspace offset inside the exported allocation (caching allocators
                     // may place it inside a larger cudaMalloc block; the handle maps the base)
  uint64_t bytes;
  int32_t rank, nranks;
  int64_t local_extent[3];
  int32_t ghost, n_gf;
  int32_t system, variant;  // neighbours must run the same kernel design (same phase count)
};

}  // namespace

struct chemora_grid_s {
  chemora_grid_desc desc;
  double params[kParams];
  Layout L;
  int64_t z0;
  char* ws;
  size_t ws_bytes;
  SetPtrs sets;
  double* dparams;          // device copy of params
  double* norm_scratch;     // kNormBlocks x len
  double* norm_out;         // len
  unsigned long long* nan_flag;
  unsigned long long* flags;  // [0] written by lo neighbour, [1] by hi neighbour
  uint64_t step;
  uint64_t epoch;
  // z-face neighbours: set bases (same SetId) of the lower / upper slab
  SetPtrs lo, hi;
  unsigned long long* lo_flag;  // where WE signal the lower neighbour (its flags[1])
  unsigned long long* hi_flag;  // where WE signal the upper neighbour (its flags[0])
  bool ipc;                     // neighbours are other processes (signal through flags)
  int cur;                      // 1: the state lives in set B (rotated by fused steps)
  std::vector<void*> opened;    // IPC mappings to close
  int variant;
  int band;                     // wave CTA band order (-1 auto; CHEMORA_WAVE_BAND)
  bool monitor;                 // NEXT-3 fused energy monitor enabled
  double* mon_partials;
  int64_t mon_n;
  double* mon_hist;             // ring of kMonHist per-step energies (device)
  double* dtab;                 // BSSN derivative table (kBssnTab x interior points) or null
  uint64_t mon_written;         // steps recorded since creation
  uint64_t mon_read;            // steps already returned by chemora_read_monitor
  double* gather;               // [nranks][kGatherLen] ring all-gather buffer (peer-read)
  double* lo_gather;            // the lower neighbour's gather buffer (IPC mapping)
  void (*barrier_fn)(void*);    // optional host barrier after every phase (shared device)
  void* barrier_user;
  // per-launch timing (chemora_set_launch_timing): events around every step launch
  bool timing;
  std::vector<cudaEvent_t> tev;  // pairs (begin, end)
  std::vector<int> tslot;        // launch slot of each pair
  size_t tn;                     // pairs recorded since the last read
};

namespace {

int n_gf_of(int system) { return system == CHEMORA_SYS_WAVE ? 5 : (system == CHEMORA_SYS_BSSN ? 25 : -1); }
int radius_of(const chemora_grid_desc& d) {
  if (d.system == CHEMORA_SYS_WAVE) return (d.fd_order == 0 ? 4 : d.fd_order) / 2;
  return 3;  // BSSN: lopsided upwind stencils reach 3 points
}

// storage ghost width: the temporally blocked wave kernels (wave_fused3.cu, orders 2, 4, 6)
// read their inputs with a halo of two stacked radius-W stencils, so those grids keep at least
// 2W ghost layers in HBM; the API's ghost width (desc.ghost) is unchanged.
int storage_ghost(const chemora_grid_desc& d) {
  const int order = d.fd_order == 0 ? 4 : d.fd_order;
  if (d.system == CHEMORA_SYS_WAVE && order <= 6) return std::max(d.ghost, order);
  return d.ghost;
}

int validate(const chemora_grid_desc* d) {
  if (!d) return fail(CHEMORA_E_INVALID, "desc is NULL");
  const int nf = n_gf_of(d->system);
  if (nf < 0) return fail(CHEMORA_E_INVALID, "unknown system " + std::to_string(d->system));
  if (d->n_gf != nf)
    return fail(CHEMORA_E_INVALID, "n_gf " + std::to_string(d->n_gf) + " does not match the system (" +
                                       std::to_string(nf) + ")");
  const int order = d->fd_order == 0 ? 4 : d->fd_order;
  if (d->system == CHEMORA_SYS_WAVE && !(order == 2 || order == 4 || order == 6 || order == 8))
    return fail(CHEMORA_E_UNSUPPORTED, "wave fd_order must be 2, 4, 6 or 8");
  if (d->system == CHEMORA_SYS_BSSN && order != 4)
    return fail(CHEMORA_E_UNSUPPORTED, "BSSN supports fd_order 4 only");
  if (d->ghost < radius_of(*d) || d->ghost > 8)
    return fail(CHEMORA_E_SHAPE, "ghost width " + std::to_string(d->ghost) +
                                     " must be >= the stencil radius " + std::to_string(radius_of(*d)) +
                                     " and <= 8");
  if (d->nranks < 1 || d->rank < 0 || d->rank >= d->nranks)
    return fail(CHEMORA_E_INVALID, "bad rank/nranks");
  for (int a = 0; a < 3; ++a) {
    if (d->extent[a] < 2 * d->ghost)
      return fail(CHEMORA_E_SHAPE, "extent[" + std::to_string(a) + "] must be >= 2*ghost");
    if (!(d->spacing[a] > 0.0) || !std::isfinite(d->spacing[a]))
      return fail(CHEMORA_E_INVALID, "spacing must be positive");
  }
  if (d->extent[0] > (int64_t(1) << 30) || d->extent[1] > (int64_t(1) << 30))
    return fail(CHEMORA_E_SHAPE, "extent too large");
  if (d->extent[2] % d->nranks)
    return fail(CHEMORA_E_SHAPE, "extent[2] must be divisible by nranks");
  if (d->extent[2] / d->nranks < 2 * d->ghost)
    return fail(CHEMORA_E_SHAPE, "local slab must have >= 2*ghost planes");
  {
    // the storage ghost width (see layout_of) must also fit
    const int gs = storage_ghost(*d);
    if (d->extent[0] < 2 * gs || d->extent[1] < 2 * gs || d->extent[2] / d->nranks < 2 * gs)
      return fail(CHEMORA_E_SHAPE, "wave grids of order 2W need >= 4W points per axis (and per slab)");
  }
  if (d->n_params < 0 || (d->n_params > 0 && !d->params) || d->n_params > kParams)
    return fail(CHEMORA_E_INVALID, "bad params");
  return CHEMORA_OK;
}

int norms_len(int system, int n_gf) { return 3 * n_gf + (system == CHEMORA_SYS_WAVE ? 1 : 0); }

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

// workspace: [sets][norm scratch][norm out][params][flags][monitor][table][gather]
constexpr int kMonHist = 1024;  // energy-monitor ring (steps)
constexpr int kMonCtas = 1024;        // max CTAs of the BSSN stage-1 launch
int mon_width(int system) { return system == CHEMORA_SYS_BSSN ? 14 : 1; }  // ring entry width
constexpr int kGatherLen = kMonHist * 14;  // doubles per rank slot of the collective gather
constexpr int kBssnTab = 136;   // BSSN derivative-table slots per point (bssn_stage.cu variant 3)
struct WsPlan {
  size_t sets, scratch, out, params, flags, mon, hist, tab, gather, total;
  int64_t mon_n;
};
WsPlan plan_ws(const Layout& L, int system, int nranks) {
  WsPlan p;
  const int len = norms_len(system, L.n_gf);
  p.sets = 0;
  size_t off = align256(sizeof(double) * (size_t)L.gfs * L.n_gf * kNumSets);
  p.scratch = off;
  off += align256(sizeof(double) * (size_t)kNormBlocks * len);
  p.out = off;
  off += align256(sizeof(double) * len);
  p.params = off;
  off += align256(sizeof(double) * kParams);
  p.flags = off;
  off += align256(sizeof(unsigned long long) * 8);  // nan flag, 2 phase flags, -, 2 scheduler words
  // NEXT-3 fused energy monitor (wave): per-CTA partials of the stage-4 launch (any CTA
  // shape 32 x BY x BZ with BY * BZ = 8) and a ring of per-step energies
  p.mon_n = 0;
  if (system == CHEMORA_SYS_WAVE) {
    const int64_t ntx = (L.nx + 31) / 32;
    p.mon_n = ntx * (L.ny * L.nz / 8 + L.ny + L.nz + 1);
  } else {
    p.mon_n = (int64_t)kMonCtas * 14;  // BSSN: per-CTA constraint partials of the stage-1 kernel
  }
  p.mon = off;
  off += align256(sizeof(double) * (size_t)p.mon_n);
  p.hist = off;
  off += align256(sizeof(double) * kMonHist * mon_width(system));
  // BSSN: HBM derivative table of the table-fission kernels, [slot][interior point]
  p.tab = off;
  if (system == CHEMORA_SYS_BSSN) off += align256(sizeof(double) * (size_t)kBssnTab * L.nx * L.ny * L.nz);
  // collective gather of per-rank results (chemora_norms & co. with nranks > 1)
  p.gather = off;
  if (nranks > 1) off += align256(sizeof(double) * (size_t)kGatherLen * nranks);
  p.total = off;
  return p;
}

Layout layout_of(const chemora_grid_desc& d) {
  return make_layout(d.extent[0], d.extent[1], d.extent[2] / d.nranks, storage_ghost(d), d.n_gf);
}

SetPtrs sets_at(char* ws, const Layout& L) {
  double* base = reinterpret_cast<double*>(ws);
  SetPtrs s;
  s.y = base + (size_t)SET_Y * L.n_gf * L.gfs + L.c0;
  s.q = base + (size_t)SET_Q * L.n_gf * L.gfs + L.c0;
  s.b = base + (size_t)SET_B * L.n_gf * L.gfs + L.c0;
  s.c = base + (size_t)SET_C * L.n_gf * L.gfs + L.c0;
  return s;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int check_grid(chemora_grid_t g) {
  if (!g) return fail(CHEMORA_E_INVALID, "grid handle is NULL");
  return CHEMORA_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// ---------------------------------------------------------------- peer signalling
// Cross-process slabs: before a phase that reads our ghosts or writes the neighbours'
// ghost planes, wait until both neighbours have finished the previous phase (their
// flags, written into OUR memory, reach epoch-1); after it, publish our epoch into theirs.
// The driver entry points are fetched through the runtime so the library has no link-time
// dependency on libcuda (it must load on the GPU-less build host).
typedef CUresult (*PFN_wait64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*PFN_write64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
PFN_wait64 g_wait64 = nullptr;
PFN_write64 g_write64 = nullptr;
typedef CUresult (*PFN_range)(CUdeviceptr*, size_t*, CUdeviceptr);
// Base of the allocation that contains p (cuMemGetAddressRange), 0 if unavailable.
uint64_t allocation_base(const void* p) {
  static PFN_range fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess || !f) return 0;
    fn = reinterpret_cast<PFN_range>(f);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, (CUdeviceptr)p) != CUDA_SUCCESS) return 0;
  return (uint64_t)base;
}

int load_stream_memops() {
  if (g_wait64 && g_write64) return CHEMORA_OK;
  cudaDriverEntryPointQueryResult q1, q2;
  void* f1 = nullptr;
  void* f2 = nullptr;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &f1, cudaEnableDefault, &q1) != cudaSuccess ||
      cudaGetDriverEntryPoint("cuStreamWriteValue64", &f2, cudaEnableDefault, &q2) != cudaSuccess ||
      !f1 || !f2)
    return fail(CHEMORA_E_PEER, "stream memory operations are unavailable");
  g_wait64 = reinterpret_cast<PFN_wait64>(f1);
  g_write64 = reinterpret_cast<PFN_write64>(f2);
  return CHEMORA_OK;
}

int phase_wait(chemora_grid_t g, cudaStream_t st) {
  if (!g->ipc || g->epoch == 0) return CHEMORA_OK;
  nvtxRangePushA("chemora phase wait");
  struct Pop { ~Pop() { nvtxRangePop(); } } pop;
  if (int rc = load_stream_memops()) return rc;
  const uint64_t want = g->epoch;  // neighbours completed phase `epoch`
  // where the device supports it, the wait also flushes outstanding remote (NVLink peer)
  // writes, so the neighbours' ghost-plane stores that preceded their flag write are visible
  // to the kernels after the wait (their flag write already carries a memory barrier)
  int can_flush = 0;
  cudaDeviceGetAttribute(&can_flush, cudaDevAttrCanFlushRemoteWrites, g->desc.device);
  const unsigned flags = CU_STREAM_WAIT_VALUE_GEQ | (can_flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0u);
  for (int f = 0; f < 2; ++f) {
    CUresult r = g_wait64((CUstream)st, (CUdeviceptr)(g->flags + f), want, flags);
    if (r != CUDA_SUCCESS) return fail(CHEMORA_E_PEER, "cuStreamWaitValue64 failed");
  }
  return CHEMORA_OK;
}
int phase_signal(chemora_grid_t g, cudaStream_t st) {
  if (!g->ipc) return CHEMORA_OK;
  if (int rc = load_stream_memops()) return rc;
  g->epoch += 1;
  CUresult r1 = g_write64((CUstream)st, (CUdeviceptr)g->lo_flag, g->epoch, 0);
  CUresult r2 = g_write64((CUstream)st, (CUdeviceptr)g->hi_flag, g->epoch, 0);
  if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS)
    return fail(CHEMORA_E_PEER, "cuStreamWriteValue64 failed");
  if (g->barrier_fn) {
    // host-ordered phases (ranks sharing one device): the phase, flag writes included, is
    // complete on this rank before any rank passes the barrier, so the next phase_wait is
    // already satisfied when it reaches the device -- no stream ever waits on another
    // process's work (chemora_set_phase_barrier)
    CUDA_TRY(cudaStreamSynchronize(st));
    g->barrier_fn(g->barrier_user);
  }
  return CHEMORA_OK;
}

// Ring all-gather of `len` doubles per rank (host src -> host out [nranks][len], rank-major),
// over the peer-mapped gather buffers, P - 1 rounds ordered by the phase flags: in round t
// rank r copies slot (r - t) mod P from its lower neighbour, which received it in round
// t - 1.  Every rank ends with the same rows in rank order, so the rank-ordered combination
// that follows is deterministic and identical everywhere.  Synchronises the stream.
int ring_allgather(chemora_grid_t g, const double* host_src, int len, double* host_out, cudaStream_t st) {
  const int P = g->desc.nranks, r = g->desc.rank;
  nvtxRangePushA("chemora ring allgather");
  struct Pop { ~Pop() { nvtxRangePop(); } } pop;
  if (len > kGatherLen) return fail(CHEMORA_E_INVALID, "gather length too large");
  if (P == 1) {
    memcpy(host_out, host_src, sizeof(double) * len);
    return CHEMORA_OK;
  }
  if (!g->ipc || !g->lo_gather) return fail(CHEMORA_E_PEER, "nranks > 1: connect the slabs with chemora_grid_connect_ipc first");
  if (int rc = phase_wait(g, st)) return rc;  // neighbours finished reading our buffer
  CUDA_TRY(cudaMemcpyAsync(g->gather + (size_t)r * kGatherLen, host_src, sizeof(double) * len,
                           cudaMemcpyHostToDevice, st));
  if (int rc = phase_signal(g, st)) return rc;
  for (int t = 1; t < P; ++t) {
    if (int rc = phase_wait(g, st)) return rc;
    const size_t slot = (size_t)((r - t + P) % P) * kGatherLen;
    CUDA_TRY(cudaMemcpyAsync(g->gather + slot, g->lo_gather + slot, sizeof(double) * len,
                             cudaMemcpyDeviceToDevice, st));
    if (int rc = phase_signal(g, st)) return rc;
  }
  for (int q = 0; q < P; ++q)
    CUDA_TRY(cudaMemcpyAsync(host_out + (size_t)q * len, g->gather + (size_t)q * kGatherLen,
                             sizeof(double) * len, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return CHEMORA_OK;
}

// Launch timing: CUDA events recorded on the launching stream around each kernel launch of
// a step (slot = which launch of the step: wave pair A/B = 0/1, else RK stage 1..4 = 0..3).
constexpr size_t kMaxTimed = 4096;
constexpr int kTimingSlots = 8;
// NVTX range names per launch slot (host-side enqueue of each phase of the step)
const char* const kPhaseName[2][4] = {{"chemora stage 1", "chemora stage 2", "chemora stage 3", "chemora stage 4"},
                                      {"chemora stages 1+2", "chemora stages 3+4", "", ""}};
cudaError_t tmark(chemora_grid_t g, int slot, bool begin, cudaStream_t st) {
  if (begin) nvtxRangePushA(kPhaseName[g->variant == 8 && g->desc.system == CHEMORA_SYS_WAVE][slot & 3]);
  else nvtxRangePop();
  if (!g->timing) return cudaSuccess;
  if (begin) {
    if (g->tn >= kMaxTimed) return cudaSuccess;  // full: later launches are not timed
    if (g->tev.size() < 2 * (g->tn + 1)) {
      for (int q = 0; q < 2; ++q) {
        cudaEvent_t e;
        cudaError_t r = cudaEventCreate(&e);
        if (r != cudaSuccess) return r;
        g->tev.push_back(e);
      }
    }
    if (g->tslot.size() < g->tn + 1) g->tslot.resize(g->tn + 1);
    g->tslot[g->tn] = slot;
    return cudaEventRecord(g->tev[2 * g->tn], st);
  }
  if (g->tn >= kMaxTimed) return cudaSuccess;
  cudaError_t r = cudaEventRecord(g->tev[2 * g->tn + 1], st);
  g->tn += 1;
  return r;
}

StageLaunch stage_args(chemora_grid_t g, double dt) {
  StageLaunch a;
  a.L = g->L;
  a.s = g->sets;
  // output set of stage s: 1 -> B, 2 -> C, 3 -> B, 4 -> y
  a.img[0] = FaceDst{g->lo.b, g->hi.b};
  a.img[1] = FaceDst{g->lo.c, g->hi.c};
  a.img[2] = FaceDst{g->lo.b, g->hi.b};
  a.img[3] = FaceDst{g->lo.y, g->hi.y};
  for (int d = 0; d < 3; ++d) a.h[d] = g->desc.spacing[d];
  a.dt = dt;
  a.fd_order = g->desc.fd_order == 0 ? 4 : g->desc.fd_order;
  a.params = g->dparams;
  for (int i = 0; i < kParams; ++i) a.hparams[i] = g->params[i];
  a.nan_flag = g->nan_flag;
  a.sched = g->nan_flag + 4;
  a.step = g->step;
  a.k_begin = 0;
  a.k_end = (int)g->L.nz;
  a.variant = g->variant;
  a.band = g->band;
  a.mon_partials = nullptr;
  a.dtab = g->dtab;
  return a;
}

cudaError_t launch_stage(chemora_grid_t g, const StageLaunch& a, int stage, cudaStream_t st) {
  return g->desc.system == CHEMORA_SYS_WAVE ? wave_stage(a, stage, st) : bssn_stage(a, stage, st);
}

// Temporally blocked wave step (wave_fused3.cu, variant 8): two kernels per step, the new
// state lands in the scratch set, which then becomes the state set.  (The round-1 pair
// designs 6 and 7 were slower in every measured configuration and are gone.)
constexpr int kVariantFused3 = 8;
bool is_fused_variant(int v) { return v == kVariantFused3; }
bool use_fused(chemora_grid_t g) {
  const int order = g->desc.fd_order == 0 ? 4 : g->desc.fd_order;
  return g->desc.system == CHEMORA_SYS_WAVE && is_fused_variant(g->variant) && order <= 6 && g->L.g >= order;
}
cudaError_t fused_pair(int variant, const StageLaunch& a, int pair, cudaStream_t st) {
  (void)variant;
  return wave_fused3_pair(a, pair, st);
}
void swap_state(chemora_grid_t g) {
  std::swap(g->sets.y, g->sets.b);
  std::swap(g->lo.y, g->lo.b);
  std::swap(g->hi.y, g->hi.b);
  g->cur ^= 1;
}

int read_nan_flag(chemora_grid_t g, cudaStream_t st) {
  unsigned long long flag = 0;
  CUDA_TRY(cudaMemcpyAsync(&flag, g->nan_flag, sizeof(flag), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (flag != ~0ull) {
    const unsigned long long step = flag / g->L.n_gf, gf = flag % g->L.n_gf;
    return fail(CHEMORA_E_NONFINITE, "non-finite value in grid function " + std::to_string(gf) +
                                         " at step " + std::to_string(step));
  }
  return CHEMORA_OK;
}

cudaMemcpy3DParms copy_params(chemora_grid_t g, int f, double* host, bool to_device, bool padded) {
  const Layout& L = g->L;
  const int gh = g->desc.ghost;  // the API's ghost width (storage may keep more, L.g)
  cudaMemcpy3DParms p;
  memset(&p, 0, sizeof(p));
  const int64_t wx = padded ? L.nx + 2 * gh : L.nx;
  const int64_t wy = padded ? L.ny + 2 * gh : L.ny;
  const int64_t wz = padded ? L.nz + 2 * gh : L.nz;
  double* dbase = g->sets.y + (size_t)f * L.gfs;  // interior origin
  double* dstart = padded ? dbase + L.idx(-gh, -gh, -gh) : dbase;
  // device pitched pointer: rows of px doubles, py rows per plane
  cudaPitchedPtr dev = make_cudaPitchedPtr(dstart, L.px * sizeof(double), wx * sizeof(double), L.py);
  double* hbase = host + (size_t)f * wx * wy * wz;
  cudaPitchedPtr hst = make_cudaPitchedPtr(hbase, wx * sizeof(double), wx * sizeof(double), wy);
  if (to_device) { p.srcPtr = hst; p.dstPtr = dev; p.kind = cudaMemcpyHostToDevice; }
  else { p.srcPtr = dev; p.dstPtr = hst; p.kind = cudaMemcpyDeviceToHost; }
  p.extent = make_cudaExtent(wx * sizeof(double), wy, wz);
  return p;
}

int halo_one(chemora_grid_t g, cudaStream_t st) {
  int rc = phase_wait(g, st);
  if (rc) return rc;
  CUDA_TRY(ghost_fill(g->L, g->sets.y, FaceDst{g->lo.y, g->hi.y}, st));
  return phase_signal(g, st);
}

}  // namespace

extern "C" {

const char* chemora_version(void) { return "chemora-b200 0.1 (sm_100a, fp64)"; }

const char* chemora_last_error(void) { return g_err.c_str(); }

int chemora_norms_len(int32_t system, int32_t n_gf) { return norms_len(system, n_gf); }

int chemora_grid_required_bytes(const chemora_grid_desc* desc, size_t* bytes) {
  int rc = validate(desc);
  if (rc) return rc;
  if (!bytes) return fail(CHEMORA_E_INVALID, "bytes is NULL");
  *bytes = plan_ws(layout_of(*desc), desc->system, desc->nranks).total;
  return CHEMORA_OK;
}

int chemora_grid_create(const chemora_grid_desc* desc, void* ws, size_t bytes, chemora_grid_t* out) {
  int rc = validate(desc);
  if (rc) return rc;
  if (!out) return fail(CHEMORA_E_INVALID, "out is NULL");
  *out = nullptr;
  if (!ws) return fail(CHEMORA_E_INVALID, "workspace is NULL");
  if (reinterpret_cast<uintptr_t>(ws) % 256) return fail(CHEMORA_E_NOMEM, "workspace must be 256-byte aligned");
  const Layout L = layout_of(*desc);
  const WsPlan P = plan_ws(L, desc->system, desc->nranks);
  if (bytes < P.total)
    return fail(CHEMORA_E_NOMEM, "workspace has " + std::to_string(bytes) + " bytes, needs " + std::to_string(P.total));
  DeviceGuard dg(desc->device);
  cudaPointerAttributes attr;
  CUDA_TRY(cudaPointerGetAttributes(&attr, ws));
  if (attr.type != cudaMemoryTypeDevice || attr.device != desc->device)
    return fail(CHEMORA_E_INVALID, "workspace is not device memory of desc->device");
  auto* g = new chemora_grid_s();
  g->desc = *desc;
  for (int i = 0; i < kParams; ++i) g->params[i] = kBenchGauge[i];
  for (int i = 0; i < desc->n_params; ++i) g->params[i] = desc->params[i];
  g->desc.params = nullptr;
  g->desc.n_params = kParams;
  g->L = L;
  g->z0 = (int64_t)desc->rank * L.nz;
  g->ws = static_cast<char*>(ws);
  g->ws_bytes = bytes;
  g->sets = sets_at(g->ws, L);
  g->norm_scratch = reinterpret_cast<double*>(g->ws + P.scratch);
  g->norm_out = reinterpret_cast<double*>(g->ws + P.out);
  g->dparams = reinterpret_cast<double*>(g->ws + P.params);
  g->dtab = g->desc.system == CHEMORA_SYS_BSSN ? reinterpret_cast<double*>(g->ws + P.tab) : nullptr;
  g->monitor = false;
  g->mon_partials = reinterpret_cast<double*>(g->ws + P.mon);
  g->mon_n = P.mon_n;
  g->mon_hist = reinterpret_cast<double*>(g->ws + P.hist);
  g->mon_written = 0;
  g->mon_read = 0;
  g->gather = reinterpret_cast<double*>(g->ws + P.gather);
  g->lo_gather = nullptr;
  g->barrier_fn = nullptr;
  g->barrier_user = nullptr;
  g->timing = false;
  g->tn = 0;
  auto* fl = reinterpret_cast<unsigned long long*>(g->ws + P.flags);
  g->nan_flag = fl;
  g->flags = fl + 1;
  g->step = 0;
  g->epoch = 0;
  // a lone slab is its own z neighbour (periodic wrap)
  g->lo = g->sets;
  g->hi = g->sets;
  g->lo_flag = g->flags + 1;
  g->hi_flag = g->flags;
  g->ipc = false;
  g->cur = 0;
  // default tiling: the temporally blocked stage pairs with register-queue z stencils for
  // wave grids of order 2, 4 and 6 (variant 8, fastest measured: order 4
  // profiles/r1_wave_design_study.md; at 512^3 order 2 7.1 vs 10.4, order 6 11.3 vs 12.4 ms/step,
  // profiles/r2_fd_orders.jsonl); order 8 (radius 4: the pair kernel's rings do not fit shared
  // memory): the persistent TMA z-march when its 32x16 tiles fill the SMs, else one thread per
  // point; BSSN: the fused per-stage kernel with the
  // derivatives on chip (variant 4: faster than the HBM-table fission, variant 3, at 192^3
  // with a fifth of its DRAM traffic, profiles/r2_bssn_summary.md)
  {
    const int order = desc->fd_order == 0 ? 4 : desc->fd_order;
    const int64_t tiles16 = ((g->L.nx + 31) / 32) * ((g->L.ny + 15) / 16);
    g->variant = desc->system == CHEMORA_SYS_BSSN ? 4 /* fused, SMEM tiles + TMEM z-windows */
               : order <= 6 ? kVariantFused3 : tiles16 >= 148 ? 4 : 0;
  }
  // plain 3-D CTA order by default: the banded order cuts DRAM reads by ~10 % but measured
  // slower under the power cap (profiles/r1_wave_summary.md); autotune may pick it (-1)
  g->band = 0;
  unsigned long long init[8] = {~0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
  cudaError_t e = cudaMemcpy(g->dparams, g->params, sizeof(g->params), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(fl, init, sizeof(init), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    delete g;
    return fail(CHEMORA_E_CUDA, std::string("grid_create: ") + cudaGetErrorString(e));
  }
  *out = g;
  return CHEMORA_OK;
}

int chemora_grid_destroy(chemora_grid_t g) {
  if (!g) return CHEMORA_OK;
  {
    DeviceGuard dg(g->desc.device);
    for (void* p : g->opened) cudaIpcCloseMemHandle(p);
    for (cudaEvent_t e : g->tev) cudaEventDestroy(e);
  }
  delete g;
  return CHEMORA_OK;
}

int chemora_grid_local(chemora_grid_t g, int64_t* ext, int64_t* z0) {
  if (int rc = check_grid(g)) return rc;
  if (ext) { ext[0] = g->L.nx; ext[1] = g->L.ny; ext[2] = g->L.nz; }
  if (z0) *z0 = g->z0;
  return CHEMORA_OK;
}

int chemora_get_kernel_variant(chemora_grid_t g, int* variant) {
  if (int rc = check_grid(g)) return rc;
  if (!variant) return fail(CHEMORA_E_INVALID, "variant is NULL");
  *variant = use_fused(g) ? g->variant : (is_fused_variant(g->variant) ? 0 : g->variant);
  return CHEMORA_OK;
}

int chemora_set_kernel_variant(chemora_grid_t g, int variant) {
  if (int rc = check_grid(g)) return rc;
  const bool ok = g->desc.system == CHEMORA_SYS_WAVE ? (variant == 0 || variant == 1 || variant == 4 || variant == kVariantFused3)
                                                    : (variant == 0 || variant == 2 || variant == 3 || variant == 4);
  if (!ok) return fail(CHEMORA_E_INVALID, "unknown kernel variant " + std::to_string(variant));
  if (g->ipc) return fail(CHEMORA_E_PEER, "the kernel design of a peer-connected slab is fixed at connect time");
  g->variant = variant;
  return CHEMORA_OK;
}

static int set_initial_nofill(chemora_grid_t g, int kind, const double* host_src, const double* kp,
                              uint64_t seed, cudaStream_t st) {
  DeviceGuard dg(g->desc.device);
  const Layout& L = g->L;
  // z-slabs in other processes: the neighbours' previous phase may still store into our
  // ghost planes, which the clear below overwrites -- wait for it first; and publish the
  // end of the clear (phase_signal below) before anyone pushes the new ghosts into us
  if (int rc = phase_wait(g, st)) return rc;
  switch (kind) {
    case CHEMORA_INIT_HOST:
    case CHEMORA_INIT_HOST_PADDED: {
      if (!host_src) return fail(CHEMORA_E_INVALID, "host_src is NULL");
      // the whole y set (ghosts included) is cleared first so unused pad is deterministic
      CUDA_TRY(cudaMemsetAsync(g->sets.y - L.c0, 0, sizeof(double) * L.gfs * L.n_gf, st));
      for (int f = 0; f < L.n_gf; ++f) {
        cudaMemcpy3DParms p = copy_params(g, f, const_cast<double*>(host_src), true,
                                          kind == CHEMORA_INIT_HOST_PADDED);
        CUDA_TRY(cudaMemcpy3DAsync(&p, st));
      }
      CUDA_TRY(cudaStreamSynchronize(st));  // host_src may be released on return
      break;
    }
    case CHEMORA_INIT_PLANE_WAVES:
    case CHEMORA_INIT_GAUSSIAN:
      if (g->desc.system != CHEMORA_SYS_WAVE) return fail(CHEMORA_E_INVALID, "init kind needs the wave system");
      /* fallthrough */
    case CHEMORA_INIT_NOISE:
    case CHEMORA_INIT_MINK_PERT:
    case CHEMORA_INIT_GAUGE_WAVE: {
      if ((kind == CHEMORA_INIT_MINK_PERT || kind == CHEMORA_INIT_GAUGE_WAVE) && g->desc.system != CHEMORA_SYS_BSSN)
        return fail(CHEMORA_E_INVALID, "MINK_PERT / GAUGE_WAVE need the BSSN system");
      InitArgs a;
      memset(&a, 0, sizeof(a));
      a.kind = kind;
      a.system = g->desc.system;
      a.seed = seed;
      a.z0 = g->z0;
      for (int d = 0; d < 3; ++d) {
        a.gext[d] = g->desc.extent[d];
        a.origin[d] = g->desc.origin[d];
        a.h[d] = g->desc.spacing[d];
      }
      if (kind == CHEMORA_INIT_GAUSSIAN) { a.kp[0] = kp ? kp[0] : 1.0; a.kp[1] = kp ? kp[1] : 0.5; }
      if (kind == CHEMORA_INIT_MINK_PERT) a.kp[0] = kp ? kp[0] : 1e-3;
      if (kind == CHEMORA_INIT_GAUGE_WAVE) {
        const double def[4] = {0.1, 1.0, 0.0, 0.0};
        for (int q = 0; q < 4; ++q) a.kp[q] = kp ? kp[q] : def[q];
        if (!(std::fabs(a.kp[0]) < 1.0) || !(a.kp[1] > 0.0))
          return fail(CHEMORA_E_INVALID, "GAUGE_WAVE needs |amp| < 1 and d > 0");
      }
      CUDA_TRY(cudaMemsetAsync(g->sets.y - L.c0, 0, sizeof(double) * L.gfs * L.n_gf, st));
      CUDA_TRY(init_interior(L, g->sets.y, a, st));
      break;
    }
    default:
      return fail(CHEMORA_E_INVALID, "unknown init kind " + std::to_string(kind));
  }
  unsigned long long nf = ~0ull;
  CUDA_TRY(cudaMemcpyAsync(g->nan_flag, &nf, sizeof(nf), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  g->step = 0;
  return phase_signal(g, st);
}

int chemora_set_initial(chemora_grid_t g, int kind, const double* host_src, const double* kp,
                        uint64_t seed, void* stream) {
  if (int rc = check_grid(g)) return rc;
  cudaStream_t st = as_stream(stream);
  if (int rc = set_initial_nofill(g, kind, host_src, kp, seed, st)) return rc;
  if (kind == CHEMORA_INIT_HOST_PADDED) return CHEMORA_OK;
  DeviceGuard dg(g->desc.device);
  return halo_one(g, st);
}

int chemora_set_initial_nofill(chemora_grid_t g, int kind, const double* host_src, const double* kp,
                               uint64_t seed, void* stream) {
  if (int rc = check_grid(g)) return rc;
  return set_initial_nofill(g, kind, host_src, kp, seed, as_stream(stream));
}

static int get_state_impl(chemora_grid_t g, double* host, void* stream, bool padded) {
  if (int rc = check_grid(g)) return rc;
  if (!host) return fail(CHEMORA_E_INVALID, "host_dst is NULL");
  DeviceGuard dg(g->desc.device);
  cudaStream_t st = as_stream(stream);
  for (int f = 0; f < g->L.n_gf; ++f) {
    cudaMemcpy3DParms p = copy_params(g, f, host, false, padded);
    CUDA_TRY(cudaMemcpy3DAsync(&p, st));
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  return read_nan_flag(g, st);
}

int chemora_debug_get_set(chemora_grid_t g, int set, double* host, void* stream) {
  if (int rc = check_grid(g)) return rc;
  if (set < 0 || set > 3 || !host) return fail(CHEMORA_E_INVALID, "bad set");
  SetPtrs saved = g->sets;
  double* p[4] = {g->sets.y, g->sets.q, g->sets.b, g->sets.c};
  g->sets.y = p[set];
  int rc = get_state_impl(g, host, stream, true);
  g->sets = saved;
  return rc;
}

int chemora_upload_state(chemora_grid_t g, const double* host, void* stream) {
  if (int rc = check_grid(g)) return rc;
  if (!host) return fail(CHEMORA_E_INVALID, "host_src is NULL");
  DeviceGuard dg(g->desc.device);
  cudaStream_t st = as_stream(stream);
  for (int f = 0; f < g->L.n_gf; ++f) {
    cudaMemcpy3DParms p = copy_params(g, f, const_cast<double*>(host), true, false);
    CUDA_TRY(cudaMemcpy3DAsync(&p, st));
  }
  CUDA_TRY(cudaMemsetAsync(g->nan_flag, 0xFF, sizeof(unsigned long long), st));  // = ~0
  return halo_one(g, st);
}

int chemora_download_state(chemora_grid_t g, double* host, void* stream) {
  if (int rc = check_grid(g)) return rc;
  if (!host) return fail(CHEMORA_E_INVALID, "host_dst is NULL");
  DeviceGuard dg(g->desc.device);
  cudaStream_t st = as_stream(stream);
  for (int f = 0; f < g->L.n_gf; ++f) {
    cudaMemcpy3DParms p = copy_params(g, f, host, false, false);
    CUDA_TRY(cudaMemcpy3DAsync(&p, st));
  }
  return CHEMORA_OK;
}

int chemora_get_state(chemora_grid_t g, double* host, void* stream) {
  return get_state_impl(g, host, stream, false);
}
int chemora_get_state_padded(chemora_grid_t g, double* host, void* stream) {
  return get_state_impl(g, host, stream, true);
}

int chemora_rhs(chemora_grid_t g, double* dst, void* stream) {
  if (int rc = check_grid(g)) return rc;
  if (!dst) return fail(CHEMORA_E_INVALID, "dev_dst is NULL");
  DeviceGuard dg(g->desc.device);
  cudaStream_t st = as_stream(stream);
  StageLaunch a = stage_args(g, 0.0);
  if (g->desc.system == CHEMORA_SYS_WAVE) CUDA_TRY(wave_rhs(a, dst, st));
  else CUDA_TRY(bssn_rhs(a, dst, st));
  return CHEMORA_OK;
}

// Fused monitors: wave -- the energy of the new state, reduced by the
// kernel that writes it (launch slot `state_slot`); BSSN -- the constraint partials of the state
// entering the step, reduced by the stage-1 kernel of the fused design (variant 4) with no extra
// pass over the state, or (other designs) by the constraint kernel before stage 1.
bool monitor_on(chemora_grid_t g) { return g->monitor && g->mon_n > 0; }
double* mon_entry(chemora_grid_t g) {
  return g->mon_hist + (g->mon_written % kMonHist) * (uint64_t)mon_width(g->desc.system);
}
cudaError_t mon_begin(chemora_grid_t g, StageLaunch& a, bool state_launch, int stage, cudaStream_t st) {
  if (!monitor_on(g)) return cudaSuccess;
  if (g->desc.system == CHEMORA_SYS_WAVE) {
    if (!state_launch) return cudaSuccess;
    a.mon_partials = g->mon_partials;
    return cudaMemsetAsync(g->mon_partials, 0, sizeof(double) * g->mon_n, st);
  }
  if (stage != 1) return cudaSuccess;
  if (g->variant == 4) {
    a.mon_partials = g->mon_partials;
    return cudaSuccess;
  }
  StageLaunch c = a;  // the state entering the step is y
  return bssn_constraints(c, nullptr, g->norm_scratch, mon_entry(g), st);
}
cudaError_t mon_end(chemora_grid_t g, const StageLaunch& a, bool state_launch, int stage, cudaStream_t st) {
  if (!monitor_on(g)) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  if (g->desc.system == CHEMORA_SYS_WAVE) {
    if (!state_launch) return cudaSuccess;
    const double vol = g->desc.spacing[0] * g->desc.spacing[1] * g->desc.spacing[2];
    e = monitor_reduce(g->mon_partials, g->mon_n, vol, mon_entry(g), st);
  } else {
    if (stage != 1) return cudaSuccess;
    if (g->variant == 4) e = bssn_constraints_reduce(g->mon_partials, bssn_fused_grid(g->L, a.k_end - a.k_begin),
                                                     mon_entry(g), st);
  }
  g->mon_written += 1;
  return e;
}

int chemora_rk4_step(chemora_grid_t g, double dt, int32_t nsteps, void* stream) {
  if (int rc = check_grid(g)) return rc;
  if (nsteps < 0 || !std::isfinite(dt)) return fail(CHEMORA_E_INVALID, "bad dt or nsteps");
  if (g->desc.nranks > 1 && !g->ipc && g->lo.y == g->sets.y)
    return fail(CHEMORA_E_PEER, "multi-slab grid is not connected");
  if (g->desc.nranks > 1 && !g->ipc)
    return fail(CHEMORA_E_PEER, "locally connected slabs step through chemora_rk4_step_multi");
  DeviceGuard dg(g->desc.device);
  cudaStream_t st = as_stream(stream);
  if (use_fused(g)) {
    for (int n = 0; n < nsteps; ++n) {
      StageLaunch a = stage_args(g, dt);
      for (int pair = 0; pair < 2; ++pair) {
        if (int rc = phase_wait(g, st)) return rc;
        CUDA_TRY(mon_begin(g, a, pair == 1, 0, st));
        CUDA_TRY(tmark(g, pair, true, st));
        CUDA_TRY(fused_pair(g->variant, a, pair, st));
        CUDA_TRY(tmark(g, pair, false, st));
        CUDA_TRY(mon_end(g, a, pair == 1, 0, st));
        if (int rc = phase_signal(g, st)) return rc;
      }
      swap_state(g);
      g->step += 1;
    }
    return CHEMORA_OK;
  }
  for (int n = 0; n < nsteps; ++n) {
    StageLaunch a = stage_args(g, dt);
    for (int s = 1; s <= 4; ++s) {
      if (int rc = phase_wait(g, st)) return rc;
      a.mon_partials = nullptr;
      CUDA_TRY(mon_begin(g, a, s == 4, s, st));
      CUDA_TRY(tmark(g, s - 1, true, st));
      CUDA_TRY(launch_stage(g, a, s, st));
      CUDA_TRY(tmark(g, s - 1, false, st));
      CUDA_TRY(mon_end(g, a, s == 4, s, st));
      if (int rc = phase_signal(g, st)) return rc;
    }
    g->step += 1;
  }
  return CHEMORA_OK;
}

int chemora_autotune(chemora_grid_t g, int32_t trials, int32_t* chosen, double* ms_out, void* stream) {
  if (int rc = check_grid(g)) return rc;
  // the trial launches store ghost images into the neighbours' sets outside the phase
  // protocol, and ranks timing independently could pick different designs: tune before
  // chemora_grid_connect_ipc (the record carries the design, connect refuses a mismatch)
  if (g->ipc) return fail(CHEMORA_E_PEER, "autotune a z-slab before chemora_grid_connect_ipc");
  if (trials < 1) trials = 3;
  DeviceGuard dg(g->desc.device);
  cudaStream_t st = as_stream(stream);
  // candidate tilings (variant, band), pruned by a footprint model:
  //   wave: one thread per point in plain order (L1/L2 reuse of every stencil operand),
  //         the persistent TMA z-march (only when its 32x16 tiles fill the SMs), and for
  //         orders 2-6 the temporally blocked stage pairs (variant 8, when the storage ghost
  //         holds their halo), else the banded L2-window order;
  //   BSSN: the fissioned one-thread-per-point kernels, the HBM-table fission and the fused
  //         per-stage kernel.
  struct Cand { int variant, band; };
  std::vector<Cand> cands;
  if (g->desc.system == CHEMORA_SYS_WAVE) {
    cands.push_back({0, 0});
    const int order = g->desc.fd_order == 0 ? 4 : g->desc.fd_order;
    const int64_t tiles = ((g->L.nx + 31) / 32) * ((g->L.ny + 15) / 16);
    if (tiles >= 148) cands.push_back({4, 0});
    if (order <= 6 && g->L.g >= order) {
      cands.push_back({kVariantFused3, 0});
    } else {
      cands.push_back({0, -1});
    }
  } else {
    cands.push_back({0, 0});
    cands.push_back({2, 0});  // fissioned one-thread-per-point kernels
    cands.push_back({3, 0});  // HBM derivative table + algebra kernels
    cands.push_back({4, 0});  // fused: SMEM plane tiles + TMEM z-windows
  }
  const int saved_v = g->variant, saved_b = g->band;
  cudaEvent_t e0, e1, e2;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  CUDA_TRY(cudaEventCreate(&e2));
  double best = 1e300;
  int besti = 0;
  for (size_t c = 0; c < cands.size(); ++c) {
    g->variant = cands[c].variant;
    g->band = cands[c].band;
    // dt = 0 and only launches that write scratch sets (B, C, Q): the state is untouched.
    // Stage-wise candidates time stages 1-3 and model stage 4 as stage 3 scaled by its
    // bytes (120 vs 112 B/pt); the temporally blocked candidate times both pair kernels
    // (its new state lands in B and is not rotated in).
    StageLaunch a = stage_args(g, 0.0);
    const bool fusedc = is_fused_variant(cands[c].variant);
    auto run = [&](float* ms3) -> cudaError_t {
      cudaError_t e = cudaSuccess;
      if (fusedc) {
        e = fused_pair(cands[c].variant, a, 0, st);
        if (e == cudaSuccess) e = fused_pair(cands[c].variant, a, 1, st);
        return e;
      }
      const int last = g->desc.system == CHEMORA_SYS_WAVE ? 3 : 1;
      for (int s = 1; s <= last && e == cudaSuccess; ++s) {
        if (s == 3 && ms3) e = cudaEventRecord(e2, st);
        if (e == cudaSuccess) e = launch_stage(g, a, s, st);
      }
      return e;
    };
    CUDA_TRY(run(nullptr));
    float msmin = 1e30f;
    for (int t = 0; t < trials; ++t) {
      float dummy = 0.f;
      CUDA_TRY(cudaEventRecord(e0, st));
      CUDA_TRY(run(&dummy));
      CUDA_TRY(cudaEventRecord(e1, st));
      CUDA_TRY(cudaEventSynchronize(e1));
      float ms = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
      if (!fusedc && g->desc.system == CHEMORA_SYS_WAVE) {
        float ms3 = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms3, e2, e1));
        ms += ms3 * 120.f / 112.f;
      }
      if (ms < msmin) msmin = ms;
    }
    if (ms_out) ms_out[c] = msmin;
    if (msmin < best) { best = msmin; besti = (int)c; }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  (void)saved_v; (void)saved_b;
  g->variant = cands[besti].variant;
  g->band = cands[besti].band;
  if (chosen) { chosen[0] = g->variant; chosen[1] = g->band; chosen[2] = (int32_t)cands.size(); }
  return CHEMORA_OK;
}

int chemora_set_monitor(chemora_grid_t g, int enable) {
  if (int rc = check_grid(g)) return rc;
  g->monitor = enable != 0;
  return CHEMORA_OK;
}

// This slab's per-step energies since the last read (no collective).
// This slab's raw per-step monitor entries since the last read (no collective): W doubles per
// step (wave: the energy h^3 sum eps; BSSN: [sum c_q^2, max |c_q|] x 7 of the local slab).
static int read_monitor_local(chemora_grid_t g, double* out, int32_t max, int32_t* count, cudaStream_t st) {
  if (int rc = check_grid(g)) return rc;
  if (!count || (max > 0 && !out)) return fail(CHEMORA_E_INVALID, "bad output buffer");
  DeviceGuard dg(g->desc.device);
  CUDA_TRY(cudaStreamSynchronize(st));
  const int W = mon_width(g->desc.system);
  const uint64_t avail = g->mon_written - g->mon_read;
  if (avail > (uint64_t)kMonHist)
    return fail(CHEMORA_E_INVALID, "monitor ring overflowed: read at least every 1024 steps");
  const int32_t n = (int32_t)(avail < (uint64_t)max ? avail : (uint64_t)(max > 0 ? max : 0));
  std::vector<double> ring((size_t)kMonHist * W);
  CUDA_TRY(cudaMemcpy(ring.data(), g->mon_hist, sizeof(double) * ring.size(), cudaMemcpyDeviceToHost));
  for (int32_t i = 0; i < n; ++i)
    for (int w = 0; w < W; ++w) out[(size_t)i * W + w] = ring[((g->mon_read + i) % kMonHist) * W + w];
  g->mon_read += n;
  *count = n;
  return read_nan_flag(g, st);
}

// Combine per-slab raw entries (rows r = 0..P-1 of n x W, slab order) into global values: sums
// (wave energy, BSSN sum c^2) added in slab order, maxima; then BSSN L2 = sqrt(h^3 sum).
static void combine_monitor(const chemora_grid_desc& d, const double* rows, int P, int32_t n, double* out) {
  const int W = mon_width(d.system);
  const double vol = d.spacing[0] * d.spacing[1] * d.spacing[2];
  for (int32_t i = 0; i < n; ++i)
    for (int w = 0; w < W; ++w) {
      const bool is_max = W > 1 && (w & 1);
      double acc = 0.0;
      for (int r = 0; r < P; ++r) {
        const double x = rows[((size_t)r * n + i) * W + w];
        acc = is_max ? std::fmax(acc, x) : acc + x;
      }
      out[(size_t)i * W + w] = (W > 1 && !is_max) ? std::sqrt(vol * acc) : acc;
    }
}

int chemora_read_monitor(chemora_grid_t g, double* out, int32_t max, int32_t* count, void* stream) {
  if (int rc = check_grid(g)) return rc;
  const int P = g->desc.nranks;
  if (P > 1 && !g->ipc)
    return fail(CHEMORA_E_PEER, "same-process slabs: read the global values with chemora_read_monitor_multi");
  cudaStream_t st = as_stream(stream);
  const int W = mon_width(g->desc.system);
  std::vector<double> mine((size_t)(max > 0 ? max : 1) * W);
  int rc = read_monitor_local(g, mine.data(), max, count, st);
  if (rc && rc != CHEMORA_E_NONFINITE) return rc;
  const int32_t n = *count;
  const std::string nonfinite = rc ? g_err : std::string();
  if (P > 1 && n > 0) {
    // collective: every rank gets the same global values (ranks step in lockstep, so n agrees)
    if ((size_t)n * W > (size_t)kGatherLen) return fail(CHEMORA_E_INVALID, "read the monitor more often");
    std::vector<double> all((size_t)n * W * P);
    DeviceGuard dg(g->desc.device);
    if (int rc1 = ring_allgather(g, mine.data(), n * W, all.data(), st)) return rc1;
    combine_monitor(g->desc, all.data(), P, n, out);
  } else if (n > 0) {
    combine_monitor(g->desc, mine.data(), 1, n, out);
  }
  if (rc) g_err = nonfinite;
  return rc;
}

int chemora_read_monitor_multi(chemora_grid_t* grids, int32_t n, double* out, int32_t max, int32_t* count,
                               void* stream) {
  if (!grids || n < 1 || !count || (max > 0 && !out)) return fail(CHEMORA_E_INVALID, "bad arguments");
  if (int rc = check_grid(grids[0])) return rc;
  const int W = mon_width(grids[0]->desc.system);
  const size_t cap = (size_t)(max > 0 ? max : 1) * W;
  std::vector<double> rows(cap * n);
  int32_t cnt0 = -1;
  int status = CHEMORA_OK;
  for (int r = 0; r < n; ++r) {
    int32_t c = 0;
    int rc = read_monitor_local(grids[r], rows.data() + cap * r, max, &c, as_stream(stream));
    if (rc && rc != CHEMORA_E_NONFINITE) return rc;
    if (rc) status = rc;
    if (cnt0 >= 0 && c != cnt0) return fail(CHEMORA_E_PEER, "slabs recorded different step counts");
    cnt0 = c;
  }
  // rows were written with stride cap; compact to n x (cnt0 x W) in slab order
  std::vector<double> packed((size_t)n * cnt0 * W);
  for (int r = 0; r < n; ++r)
    for (size_t q = 0; q < (size_t)cnt0 * W; ++q) packed[(size_t)r * cnt0 * W + q] = rows[cap * r + q];
  if (cnt0 > 0) combine_monitor(grids[0]->desc, packed.data(), n, cnt0, out);
  *count = cnt0;
  return status;
}

int chemora_set_launch_timing(chemora_grid_t g, int enable) {
  if (int rc = check_grid(g)) return rc;
  g->timing = enable != 0;
  g->tn = 0;
  return CHEMORA_OK;
}

int chemora_read_launch_timing(chemora_grid_t g, double* ms_sum, int32_t* counts, void* stream) {
  if (int rc = check_grid(g)) return rc;
  if (!ms_sum || !counts) return fail(CHEMORA_E_INVALID, "output is NULL");
  DeviceGuard dg(g->desc.device);
  CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
  for (int s = 0; s < kTimingSlots; ++s) { ms_sum[s] = 0.0; counts[s] = 0; }
  for (size_t i = 0; i < g->tn; ++i) {
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, g->tev[2 * i], g->tev[2 * i + 1]));
    const int s = g->tslot[i];
    if (s >= 0 && s < kTimingSlots) { ms_sum[s] += ms; counts[s] += 1; }
  }
  g->tn = 0;
  return CHEMORA_OK;
}

int chemora_set_phase_barrier(chemora_grid_t g, void (*fn)(void*), void* user) {
  if (int rc = check_grid(g)) return rc;
  g->barrier_fn = fn;
  g->barrier_user = user;
  return CHEMORA_OK;
}

int chemora_rk4_step_multi(chemora_grid_t* grids, int32_t n, double dt, int32_t nsteps, void* stream) {
  if (!grids || n < 1) return fail(CHEMORA_E_INVALID, "bad grid list");
  for (int r = 0; r < n; ++r)
    if (int rc = check_grid(grids[r])) return rc;
  if (nsteps < 0 || !std::isfinite(dt)) return fail(CHEMORA_E_INVALID, "bad dt or nsteps");
  DeviceGuard dg(grids[0]->desc.device);
  cudaStream_t st = as_stream(stream);
  bool fused = true;
  for (int r = 0; r < n; ++r) fused = fused && use_fused(grids[r]);
  // per-slab fused monitors (the global values combine the slabs', chemora_read_monitor_multi)
  for (int step = 0; step < nsteps; ++step) {
    if (fused) {
      for (int pair = 0; pair < 2; ++pair)
        for (int r = 0; r < n; ++r) {
          StageLaunch a = stage_args(grids[r], dt);
          CUDA_TRY(mon_begin(grids[r], a, pair == 1, 0, st));
          CUDA_TRY(fused_pair(grids[r]->variant, a, pair, st));
          CUDA_TRY(mon_end(grids[r], a, pair == 1, 0, st));
        }
      for (int r = 0; r < n; ++r) swap_state(grids[r]);
    } else {
      for (int s = 1; s <= 4; ++s)
        for (int r = 0; r < n; ++r) {
          StageLaunch a = stage_args(grids[r], dt);
          CUDA_TRY(mon_begin(grids[r], a, s == 4, s, st));
          CUDA_TRY(launch_stage(grids[r], a, s, st));
          CUDA_TRY(mon_end(grids[r], a, s == 4, s, st));
        }
    }
    for (int r = 0; r < n; ++r) grids[r]->step += 1;
  }
  return CHEMORA_OK;
}

int chemora_halo_exchange(chemora_grid_t g, void* stream) {
  if (int rc = check_grid(g)) return rc;
  DeviceGuard dg(g->desc.device);
  return halo_one(g, as_stream(stream));
}

int chemora_halo_exchange_multi(chemora_grid_t* grids, int32_t n, void* stream) {
  if (!grids || n < 1) return fail(CHEMORA_E_INVALID, "bad grid list");
  DeviceGuard dg(grids[0]->desc.device);
  cudaStream_t st = as_stream(stream);
  // per slab: x, y fill then the z push into the neighbours' ghost planes (a push only
  // writes z-ghost planes, which no other slab's x/y fill touches)
  for (int r = 0; r < n; ++r) {
    chemora_grid_t g = grids[r];
    CUDA_TRY(ghost_fill(g->L, g->sets.y, FaceDst{g->lo.y, g->hi.y}, st));
  }
  return CHEMORA_OK;
}

int chemora_norms_partial(chemora_grid_t g, double* out, void* stream) {
  if (int rc = check_grid(g)) return rc;
  if (!out) return fail(CHEMORA_E_INVALID, "out is NULL");
  DeviceGuard dg(g->desc.device);
  cudaStream_t st = as_stream(stream);
  const int len = norms_len(g->desc.system, g->L.n_gf);
  CUDA_TRY(norms_partial(g->L, g->sets.y, g->desc.system, g->norm_scratch, g->norm_out, st));
  CUDA_TRY(cudaMemcpyAsync(out, g->norm_out, sizeof(double) * len, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return read_nan_flag(g, st);
}

int chemora_norms_combine(const chemora_grid_desc* d, const double* partials, int32_t nranks, double* out) {
  if (!d || !partials || !out || nranks < 1) return fail(CHEMORA_E_INVALID, "bad arguments");
  const int nf = n_gf_of(d->system);
  if (nf < 0) return fail(CHEMORA_E_INVALID, "unknown system");
  const int len = norms_len(d->system, nf);
  const double vol = d->spacing[0] * d->spacing[1] * d->spacing[2];
  for (int v = 0; v < len; ++v) {
    double acc = 0.0;
    for (int r = 0; r < nranks; ++r) {
      const double x = partials[(size_t)r * len + v];
      acc = (v % 3 == 1 && v < 3 * nf) ? std::fmax(acc, x) : acc + x;
    }
    if (v < 3 * nf && v % 3 == 0) out[v] = std::sqrt(vol * acc);
    else if (v < 3 * nf && v % 3 == 1) out[v] = acc;
    else out[v] = vol * acc;
  }
  return CHEMORA_OK;
}

int chemora_norms(chemora_grid_t g, double* out, void* stream) {
  if (int rc = check_grid(g)) return rc;
  if (!out) return fail(CHEMORA_E_INVALID, "out is NULL");
  const int len = norms_len(g->desc.system, g->L.n_gf), P = g->desc.nranks;
  std::vector<double> part(len), all((size_t)len * P);
  int rc = chemora_norms_partial(g, part.data(), stream);
  if (rc && rc != CHEMORA_E_NONFINITE) return rc;
  const std::string nonfinite = rc ? g_err : std::string();
  DeviceGuard dg(g->desc.device);
  if (int rc1 = ring_allgather(g, part.data(), len, all.data(), as_stream(stream))) return rc1;
  int rc2 = chemora_norms_combine(&g->desc, all.data(), P, out);
  if (rc && !rc2) g_err = nonfinite;
  return rc ? rc : rc2;
}

int chemora_constraints(chemora_grid_t g, double* fields, double* out, void* stream) {
  if (int rc = check_grid(g)) return rc;
  if (g->desc.system != CHEMORA_SYS_BSSN) return fail(CHEMORA_E_UNSUPPORTED, "constraints: BSSN only");
  DeviceGuard dg(g->desc.device);
  cudaStream_t st = as_stream(stream);
  StageLaunch a = stage_args(g, 0.0);
  CUDA_TRY(bssn_constraints(a, fields, g->norm_scratch, g->norm_out, st));
  if (!out) return CHEMORA_OK;
  CUDA_TRY(cudaMemcpyAsync(out, g->norm_out, sizeof(double) * 14, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return read_nan_flag(g, st);
}

int chemora_constraint_norms_combine(const chemora_grid_desc* d, const double* partials, int32_t nranks,
                                     double* out) {
  if (!d || !partials || !out || nranks < 1) return fail(CHEMORA_E_INVALID, "bad arguments");
  const double vol = d->spacing[0] * d->spacing[1] * d->spacing[2];
  for (int q = 0; q < 7; ++q) {
    double s = 0.0, m = 0.0;
    for (int r = 0; r < nranks; ++r) {
      s += partials[(size_t)r * 14 + 2 * q];
      m = std::fmax(m, partials[(size_t)r * 14 + 2 * q + 1]);
    }
    out[2 * q] = std::sqrt(vol * s);
    out[2 * q + 1] = m;
  }
  return CHEMORA_OK;
}

int chemora_constraint_norms(chemora_grid_t g, double* out, void* stream) {
  if (int rc = check_grid(g)) return rc;
  if (!out) return fail(CHEMORA_E_INVALID, "out is NULL");
  const int P = g->desc.nranks;
  double part[14];
  int rc = chemora_constraints(g, nullptr, part, stream);
  if (rc && rc != CHEMORA_E_NONFINITE) return rc;
  const std::string nonfinite = rc ? g_err : std::string();
  std::vector<double> all((size_t)14 * P);
  DeviceGuard dg(g->desc.device);
  if (int rc1 = ring_allgather(g, part, 14, all.data(), as_stream(stream))) return rc1;
  int rc2 = chemora_constraint_norms_combine(&g->desc, all.data(), P, out);
  if (rc && !rc2) g_err = nonfinite;
  return rc ? rc : rc2;
}

int chemora_grid_connect_local(chemora_grid_t* grids, int32_t n) {
  if (!grids || n < 1) return fail(CHEMORA_E_INVALID, "bad grid list");
  for (int r = 0; r < n; ++r) {
    if (int rc = check_grid(grids[r])) return rc;
    if (grids[r]->desc.rank != r || grids[r]->desc.nranks != n)
      return fail(CHEMORA_E_PEER, "grids[r] must have rank r of n");
    if (grids[r]->desc.device != grids[0]->desc.device)
      return fail(CHEMORA_E_PEER, "local slabs must share one device");
    if (grids[r]->L.gfs != grids[0]->L.gfs || grids[r]->L.nz != grids[0]->L.nz)
      return fail(CHEMORA_E_PEER, "slabs have different layouts");
  }
  for (int r = 0; r < n; ++r) {
    chemora_grid_t g = grids[r];
    g->lo = grids[(r + n - 1) % n]->sets;
    g->hi = grids[(r + 1) % n]->sets;
    g->ipc = false;
  }
  return CHEMORA_OK;
}

int chemora_peer_record_size(size_t* bytes) {
  if (!bytes) return fail(CHEMORA_E_INVALID, "bytes is NULL");
  *bytes = sizeof(PeerRecord);
  return CHEMORA_OK;
}

int chemora_grid_export_peer(chemora_grid_t g, void* rec_out) {
  if (int rc = check_grid(g)) return rc;
  if (!rec_out) return fail(CHEMORA_E_INVALID, "record_out is NULL");
  DeviceGuard dg(g->desc.device);
  PeerRecord rec;
  memset(&rec, 0, sizeof(rec));
  CUDA_TRY(cudaIpcGetMemHandle(&rec.handle, g->ws));
  const uint64_t base = allocation_base(g->ws);
  if (!base) return fail(CHEMORA_E_PEER, "cuMemGetAddressRange failed for the workspace");
  rec.offset = (uint64_t)(uintptr_t)g->ws - base;
  rec.bytes = g->ws_bytes;
  rec.rank = g->desc.rank;
  rec.nranks = g->desc.nranks;
  rec.local_extent[0] = g->L.nx; rec.local_extent[1] = g->L.ny; rec.local_extent[2] = g->L.nz;
  rec.ghost = g->L.g;
  rec.n_gf = g->L.n_gf;
  rec.system = g->desc.system;
  rec.variant = g->variant;
  memcpy(rec_out, &rec, sizeof(rec));
  return CHEMORA_OK;
}

int chemora_grid_connect_ipc(chemora_grid_t g, const void* rlo, const void* rhi) {
  if (int rc = check_grid(g)) return rc;
  if (!rlo || !rhi) return fail(CHEMORA_E_INVALID, "record is NULL");
  PeerRecord lo, hi;
  memcpy(&lo, rlo, sizeof(lo));
  memcpy(&hi, rhi, sizeof(hi));
  const int n = g->desc.nranks, r = g->desc.rank;
  if (lo.rank != (r + n - 1) % n || hi.rank != (r + 1) % n || lo.nranks != n || hi.nranks != n)
    return fail(CHEMORA_E_PEER, "records are not this rank's ring neighbours");
  for (const PeerRecord* p : {&lo, &hi})
    if (p->local_extent[0] != g->L.nx || p->local_extent[1] != g->L.ny ||
        p->local_extent[2] != g->L.nz || p->ghost != g->L.g || p->n_gf != g->L.n_gf)
      return fail(CHEMORA_E_PEER, "neighbour layout differs");
  for (const PeerRecord* p : {&lo, &hi})
    if (p->system != g->desc.system || p->variant != g->variant)
      return fail(CHEMORA_E_PEER, "neighbour runs a different system or kernel design (variant " +
                                      std::to_string(p->variant) + " vs " + std::to_string(g->variant) + ")");
  DeviceGuard dg(g->desc.device);
  const WsPlan P = plan_ws(g->L, g->desc.system, g->desc.nranks);
  auto open = [&](const PeerRecord& rec, char** base) -> int {
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, rec.handle, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(CHEMORA_E_PEER, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    g->opened.push_back(p);
    *base = static_cast<char*>(p) + rec.offset;
    return CHEMORA_OK;
  };
  char* blo = nullptr;
  char* bhi = nullptr;
  if (int rc = open(lo, &blo)) return rc;
  if (n == 2) bhi = blo;  // both faces go to the same peer
  else if (int rc = open(hi, &bhi)) return rc;
  g->lo = sets_at(blo, g->L);
  if (g->cur) {  // state/scratch sets already rotated by fused steps (neighbours in lockstep)
    SetPtrs t = sets_at(blo, g->L);
    g->lo.y = t.b;
    g->lo.b = t.y;
  }
  g->hi = sets_at(bhi, g->L);
  if (g->cur) {
    SetPtrs t = sets_at(bhi, g->L);
    g->hi.y = t.b;
    g->hi.b = t.y;
  }
  // we signal the lower neighbour in its flags[1] ("from hi") and the upper in flags[0]
  g->lo_flag = reinterpret_cast<unsigned long long*>(blo + P.flags) + 2;
  g->hi_flag = reinterpret_cast<unsigned long long*>(bhi + P.flags) + 1;
  g->lo_gather = reinterpret_cast<double*>(blo + P.gather);
  g->ipc = true;
  g->epoch = 0;
  return CHEMORA_OK;
}

}  // extern "C"
