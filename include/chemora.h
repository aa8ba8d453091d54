/* chemora.h -- C ABI of the B200-native fused RK4 finite-difference stencil library.
 *
 * The hot path of Chemora's method (arXiv:1410.1764, /root/reference/PAPER.md): a
 * generated finite-difference loop kernel that evaluates the right-hand side of a system
 * of PDE grid functions on a 3-D Cartesian grid with ghost zones (PAPER.md:320-347,
 * Eq. 1 and the Sec. 3 loop listing), stepped in time by a Runge-Kutta method
 * (PAPER.md:209-219), with the grid decomposed across devices by the driver
 * (PAPER.md:200-207).  Every call below names the passage that defines its operation.
 *
 * Conventions
 *  - fp64 everywhere.  Grid functions ("GF") are stored structure-of-arrays,
 *    [gf][z][y][x] with x contiguous.  Host arrays passed in or out are INTERIOR-only,
 *    [gf][Nz_local][Ny][Nx] (or padded [gf][Nz_local+2g][Ny+2g][Nx+2g] where stated).
 *  - Device memory is OWNED BY THE CALLER: chemora_grid_required_bytes() says how much,
 *    the caller allocates it (e.g. torch.empty(bytes, dtype=uint8, device=cuda)) and passes
 *    it to chemora_grid_create(); it must outlive the handle and be 256-byte aligned.
 *  - Streams are borrowed (cudaStream_t passed as void*; NULL = legacy default stream).
 *    Calls ENQUEUE work on the stream and return; device faults and non-finite values
 *    surface at the next synchronising call (chemora_get_state*, chemora_norms*).  The
 *    calls on one handle must be ordered (one stream, or streams ordered by events): the
 *    handle's workspace holds its state sets, flags and the kernels' work-item counter.
 *    Different handles may run concurrently on different streams.
 *  - Every function returns a chemora_status; on failure a thread-local message is
 *    available from chemora_last_error().  No function aborts the process.
 *  - Boundary: periodic on all axes (reading R9).  With nranks > 1
 *    the global grid is split into z-slabs of extent[2]/nranks planes (rank r owns global
 *    planes [r*Nz/P, (r+1)*Nz/P)); x and y stay whole on every rank.
 */
#ifndef CHEMORA_H
#define CHEMORA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct chemora_grid_s* chemora_grid_t; /* opaque handle */

enum chemora_status {
  CHEMORA_OK = 0,
  CHEMORA_E_INVALID = 1,     /* bad argument (NULL pointer, wrong n_gf, unknown kind ...) */
  CHEMORA_E_SHAPE = 2,       /* extents / ghost width violate the grid invariants          */
  CHEMORA_E_NOMEM = 3,       /* workspace too small or misaligned                          */
  CHEMORA_E_CUDA = 4,        /* CUDA runtime/driver error (message has the CUDA string)    */
  CHEMORA_E_PEER = 5,        /* multi-rank connectivity error                              */
  CHEMORA_E_NONFINITE = 6,   /* NaN/Inf produced by a step (message names GF and step)     */
  CHEMORA_E_UNSUPPORTED = 7  /* valid request this build does not implement                */
};

/* PDE systems.  WAVE: the first-order scalar wave equation, Eq. 1 (PAPER.md:320-327,
 * Fig. 1), 5 GFs in order u, rho, v1, v2, v3.
 * BSSN: the 25-GF BSSN-like Einstein system of SURVEY.md App. A (PAPER.md:686-688 says only
 * "the Einstein equations ... several thousand floating point operations"; R7),
 * GFs in the order phi, gt11 gt12 gt13 gt22 gt23 gt33, trK, At11..At33, Xt1..3, alpha, A,
 * beta1..3, B1..3. */
enum chemora_system { CHEMORA_SYS_WAVE = 1, CHEMORA_SYS_BSSN = 2 };

/* Initial-data kinds for chemora_set_initial (Fig. 1 "Init"). */
enum chemora_init {
  CHEMORA_INIT_HOST = 0,        /* host_src: interior [gf][Nz_local][Ny][Nx]; ghosts filled  */
  CHEMORA_INIT_HOST_PADDED = 1, /* host_src: padded [gf][Nz_local+2g][Ny+2g][Nx+2g]; ghosts
                                   taken AS GIVEN (no fill) -- for polynomial tests          */
  CHEMORA_INIT_PLANE_WAVES = 2, /* wave: the PW3 superposition of DESIGN.md §Inputs           */
  CHEMORA_INIT_GAUSSIAN = 3,    /* wave: rho = A exp(-(r/W)^2/2) at the domain centre;
                                   kind_params = {A, W} or NULL for {1, 0.5}                 */
  CHEMORA_INIT_NOISE = 4,       /* every GF = SplitMix64(seed ^ (gf<<40 + I)) -> [-1,1),
                                   I = global interior index i + Nx (j + Ny k)               */
  CHEMORA_INIT_MINK_PERT = 5,   /* BSSN: flat + seeded sines, kind_params = {eps} or NULL   */
  CHEMORA_INIT_GAUGE_WAVE = 6   /* BSSN: the gauge-wave exact solution at time t (SURVEY.md
                                   App. A.3), H = 1 - amp sin(2 pi (x + s t - t)/d),
                                   constant shift beta^x = s; kind_params = {amp, d, s, t} or
                                   NULL for {0.1, 1, 0, 0}; needs |amp| < 1, d > 0        */
};

/* Grid descriptor (SPEC.md:415-418 UniformGrid). */
typedef struct {
  int32_t system;       /* enum chemora_system                                          */
  int32_t ghost;        /* ghost width g; must be >= the stencil radius (2 wave, 3 BSSN)  */
  int32_t n_gf;         /* number of grid functions; must be 5 (WAVE) or 25 (BSSN)       */
  int32_t device;       /* CUDA device ordinal the workspace lives on                    */
  int64_t extent[3];    /* GLOBAL interior extents Nx, Ny, Nz; each >= 2g; Nz % nranks == 0,
                           and Nz/nranks >= 2g                                           */
  double origin[3];     /* x_i = origin + i * h                            */
  double spacing[3];    /* h per axis                                                     */
  int32_t rank;         /* z-slab index of this handle, 0 <= rank < nranks               */
  int32_t nranks;       /* number of z-slabs (processes or local slabs)                  */
  int32_t fd_order;     /* accuracy order of the centered stencils: 0 or 4 (default), or
                           2, 6, 8 for WAVE ("arbitrary order ... run-time
                           option"); requires ghost >= fd_order/2                         */
  int32_t n_params;     /* number of entries in params                                   */
  const double* params; /* BSSN gauge parameters F_alpha, n_alpha, L, eta_alpha,
                           c_alpha_adv, C_beta, p_beta, S_B, eta, c_beta_adv (App. A.3);
                           NULL = the benchmark gauge {2,1,1,0,1,0.75,0,1,1,1}. Copied. */
} chemora_grid_desc;

/* Library version string (static storage). */
const char* chemora_version(void);

/* Thread-local text describing the last non-OK return on this thread. */
const char* chemora_last_error(void);

/* Bytes of device workspace the grid needs (4 state sets of n_gf padded arrays: the
 * y/Q/B/C scheme of DESIGN.md §RK4, padded with max(ghost, fd_order) layers for wave orders
 * 2-6 (the stage-pair kernels' halo) and ghost layers otherwise, plus reduction scratch and
 * flags; for BSSN also the
 * derivative table of kernel variant 3: 136 doubles per local interior point, e.g. 7.7 GB
 * at 192^3).  Validates desc. */
int chemora_grid_required_bytes(const chemora_grid_desc* desc, size_t* bytes);

/* Create a grid handle over a caller-owned device workspace of >= required bytes.
 * Does not initialise the state (call chemora_set_initial). */
int chemora_grid_create(const chemora_grid_desc* desc, void* dev_workspace, size_t bytes,
                        chemora_grid_t* out);

/* Destroy the handle (does not free the caller's workspace).  NULL is a no-op. */
int chemora_grid_destroy(chemora_grid_t grid);

/* Local geometry: local interior extents and the global z index of local plane 0. */
int chemora_grid_local(chemora_grid_t grid, int64_t* local_extent3, int64_t* z0);

/* Set the state vector y (Fig. 1 "Init").  kind = enum chemora_init.
 * HOST / HOST_PADDED copy from host_src (pageable or pinned; the call waits for the copy
 * to be read), the analytic kinds are generated on the device from GLOBAL coordinates.
 * Every kind except HOST_PADDED ends with chemora_halo_exchange (collective when
 * nranks > 1).  Resets the step counter and the non-finite flag. */
int chemora_set_initial(chemora_grid_t grid, int kind, const double* host_src,
                        const double* kind_params, uint64_t seed, void* stream);

/* Copy the local interior of y to host_dst [gf][Nz_local][Ny][Nx]; synchronises the stream.
 * Returns CHEMORA_E_NONFINITE if a previous step produced NaN/Inf (data still copied). */
int chemora_get_state(chemora_grid_t grid, double* host_dst, void* stream);

/* Stream-ordered state transfer for pipelined host I/O (several grids / streams in flight):
 * enqueue the copy of the local interior [gf][Nz_local][Ny][Nx] from / to PINNED host memory
 * on `stream` and return without synchronising; the caller keeps the host buffer alive and
 * unmodified until the stream has passed this point.  chemora_upload_state then fills the
 * ghosts (chemora_halo_exchange, collective when nranks > 1) and clears the non-finite flag;
 * unlike chemora_set_initial it does not reset the step counter or clear the pad.  Non-finite
 * values surface at the next chemora_get_state / chemora_norms*. */
int chemora_upload_state(chemora_grid_t grid, const double* host_src, void* stream);
int chemora_download_state(chemora_grid_t grid, double* host_dst, void* stream);

/* As chemora_get_state but padded [gf][Nz_local+2g][Ny+2g][Nx+2g], ghosts included. */
int chemora_get_state_padded(chemora_grid_t grid, double* host_dst, void* stream);

/* k = F(y) at every local interior point, ghosts of y used as they are (SPEC.md:442-450
 * apply_kernel; the RHS of Eq. 1 or App. A).  dev_dst: device, n_gf x local interior,
 * [gf][z][y][x], caller-owned. */
int chemora_rhs(chemora_grid_t grid, double* dev_dst, void* stream);

/* Advance y by nsteps classical RK4 steps of size dt.
 * Each step is 4 fused stage kernels; each stage evaluates the RHS of its input, applies
 * the RK4 update, writes the periodic ghost images of its output, and (nranks > 1) stores
 * its boundary planes into the neighbours' ghost planes (the halo exchange, PAPER.md:
 * 201-204, 346).  On return (stream-ordered) y's ghosts are consistent.  nranks > 1 with
 * peers connected through chemora_grid_connect_ipc is collective over all ranks. */
int chemora_rk4_step(chemora_grid_t grid, double dt, int32_t nsteps, void* stream);

/* Same, for n local slabs of ONE global grid living in this process (all on one device,
 * connected with chemora_grid_connect_local); stages are interleaved slab by slab on
 * the one stream.  This is the single-device emulation of the multi-GPU path. */
int chemora_rk4_step_multi(chemora_grid_t* grids, int32_t n, double dt, int32_t nsteps,
                           void* stream);

/* Periodic ghost fill of y: x and y locally, z by wrap (nranks == 1) or by storing the
 * boundary planes into the neighbours' ghost planes (nranks > 1) (
 * SPEC.md:433-441 sync_ghosts).  Collective when nranks > 1. */
int chemora_halo_exchange(chemora_grid_t grid, void* stream);
int chemora_halo_exchange_multi(chemora_grid_t* grids, int32_t n, void* stream);

/* Local reduction partials of y over the local interior (SPEC.md:469-477 reduce; Fig. 1
 * "Energy"): out[3v+0] = sum f^2, out[3v+1] = max|f|, out[3v+2] = sum f
 * for v < n_gf, then (WAVE) out[3 n_gf] = sum 1/2 (rho^2 + v.v).  Deterministic order.
 * Synchronises the stream.  Returns CHEMORA_E_NONFINITE as chemora_get_state.  Not
 * collective (the building block of chemora_norms). */
int chemora_norms_partial(chemora_grid_t grid, double* host_out, void* stream);

/* Combine per-rank partials (rank-major, nranks x chemora_norms_len doubles) in rank order
 * into L2 = sqrt(h^3 sum f^2), Linf, h^3 sum f (and the energy h^3 sum eps). */
int chemora_norms_combine(const chemora_grid_desc* desc, const double* partials,
                          int32_t nranks, double* out);

/* Number of doubles chemora_norms / chemora_norms_partial write: 3 n_gf (+1 for WAVE). */
int chemora_norms_len(int32_t system, int32_t n_gf);

/* Global norms of y (SPEC.md:469-477 reduce; "Energy"): host_out
 * (chemora_norms_len doubles) = per GF L2 = sqrt(h^3 sum f^2), Linf = max|f|, h^3 sum f, then
 * (WAVE) the energy h^3 sum 1/2 (rho^2 + v.v), over the WHOLE grid.  nranks > 1: COLLECTIVE
 * over all slabs of a chemora_grid_connect_ipc ring (every rank calls it at the same point
 * of its call sequence): the per-rank partials are all-gathered through the peer-mapped
 * workspaces (P - 1 ring rounds ordered by the same epoch flags as the step) and combined
 * in rank order, so every rank returns the identical, deterministic result.  Synchronises.
 * Returns CHEMORA_E_NONFINITE (after filling host_out) if this rank's state holds NaN/Inf;
 * CHEMORA_E_PEER if nranks > 1 and the slab is not connected. */
int chemora_norms(chemora_grid_t grid, double* host_out, void* stream);

/* ---- multi-slab connectivity (z-slab ring, rank r's neighbours are r-1 and r+1 mod P)
 *
 * The planned NCCL bootstrap (chemora_get_unique_id + an ncclUniqueId in the descriptor,
 * SURVEY.md §8(b)) is replaced by peer memory: the halo exchange is
 * fused into the stage kernels, which store their boundary planes straight into the
 * neighbours' ghost planes through CUDA-IPC mappings of the neighbours' workspaces, and the
 * phases are ordered by stream memory operations on epoch flags in the workspaces
 * (DESIGN.md §6).  The only bootstrap data is the opaque per-rank peer record below, which
 * the caller exchanges (e.g. torch.distributed.all_gather_object); no NCCL communicator
 * exists.  The collective calls (chemora_rk4_step, chemora_halo_exchange,
 * chemora_set_initial, chemora_upload_state, chemora_norms, chemora_constraint_norms,
 * chemora_read_monitor) must be made by every rank in the same order. */

/* Same-process slabs (emulation on one device): grids[r] has rank r of n. */
int chemora_grid_connect_local(chemora_grid_t* grids, int32_t n);

/* Cross-process: size of the opaque per-rank peer record, export this rank's record
 * (cudaIpc handle of the workspace), and connect to the lower and upper neighbours'
 * records (exchanged by the caller, e.g. torch.distributed.all_gather_object). */
int chemora_peer_record_size(size_t* bytes);
int chemora_grid_export_peer(chemora_grid_t grid, void* record_out);
int chemora_grid_connect_ipc(chemora_grid_t grid, const void* record_lo, const void* record_hi);
/* (The record also carries the system and kernel design; connect fails with CHEMORA_E_PEER
 * if a neighbour's differ -- the step's phase count depends on the design.  After connect
 * chemora_set_kernel_variant and chemora_autotune are refused.) */

/* Optional host barrier after every phase of the cross-process protocol: fn(user) is called
 * (after synchronising the stream) at the end of each phase, and must return only when every
 * rank has reached the same point (e.g. a torch.distributed gloo barrier).  The stream waits
 * of the next phase are then already satisfied when they reach the device, so no stream ever
 * waits on another process's work -- required when several ranks share ONE device (their
 * contexts are time-sliced), and a debugging aid otherwise.  fn = NULL restores the default
 * (device-side ordering only). */
int chemora_set_phase_barrier(chemora_grid_t grid, void (*fn)(void* user), void* user);

/* ---- analysis and tuning */

/* Fused monitors.  WAVE: energy (Fig. 1 "Energy" eps = 1/2 (rho^2 + delta^ij v_i v_j),
 * PAPER.md:642-644): when enabled, the kernel of every chemora_rk4_step(_multi) step that
 * writes the new state (the stage-4 kernel, or the stage-pair kernel B of the temporally
 * blocked path) also reduces E = h^3 sum eps of that state over the LOCAL slab
 * (deterministic partials per CTA or per work item + a fixed-order sum) -- no extra HBM pass
 * over the state.
 * BSSN: the constraint monitors H, M^i, G^i (R16) of the state
 * entering every step, reduced by the step's stage-1 kernel (kernel design 4: from the
 * derivatives it computes anyway; other designs: the constraint kernel before stage 1).
 * Read with chemora_read_monitor (global values, collective for nranks > 1) or
 * chemora_read_monitor_multi (same-process slabs). */
int chemora_set_monitor(chemora_grid_t grid, int enable);

/* Copy the monitor values of up to max steps recorded since the last read (oldest first) to
 * out; *count receives the number of steps.  WAVE: one double per step, the energy after the
 * step.  BSSN: 14 doubles per step, [L2 = sqrt(h^3 sum c^2), Linf] of H, M1..3, G1..3 (the
 * constraints of chemora_constraints) of the state ENTERING the step -- computed by the
 * fused stage-1 kernel of kernel design 4 from the derivatives it already holds on chip (no
 * extra pass over the state; other designs run the constraint kernel before stage 1).
 * Synchronises the stream.  The device ring holds 1024 steps; reading less often is an error
 * (CHEMORA_E_INVALID).  nranks > 1 (IPC ring): COLLECTIVE, the values are global (the slabs'
 * partials all-gathered and combined in rank order), identical on every rank. */
int chemora_read_monitor(chemora_grid_t grid, double* out, int32_t max, int32_t* count,
                         void* stream);
/* The same for n same-process slabs (chemora_grid_connect_local): slab values added in slab
 * order. */
int chemora_read_monitor_multi(chemora_grid_t* grids, int32_t n, double* out, int32_t max,
                               int32_t* count, void* stream);

/* BSSN constraint monitors ("constraint equations"; SURVEY.md §8(f)
 * NEXT-3; reading R16), from the current state y with the RHS's 4th-order
 * stencils (ghosts of y used as they are -- consistent after every call that returns y):
 *   H   = e^{-4 phi} gt^ij (R~_ij + R^phi_ij) + 2/3 K^2 - At_ij At^ij
 *   M^i = d_j At^ij + Gt^i_jk At^jk + 6 At^ij d_j phi - 2/3 gt^ij d_j K
 *   G^i = Xt^i - gt^jk Gt^i_jk
 * dev_fields (device, nullable): 7 x local interior, [H, M1, M2, M3, G1, G2, G3][z][y][x],
 * caller-owned.  host_out (nullable, 14 doubles): per constraint q, the local partials
 * host_out[2q] = sum c_q^2 and host_out[2q+1] = max |c_q| in a fixed (deterministic) order;
 * with nranks == 1, chemora_constraint_norms turns them into L2 = sqrt(h^3 sum) and Linf.
 * BSSN only (CHEMORA_E_UNSUPPORTED otherwise).  Synchronises the stream when host_out is
 * given. */
int chemora_constraints(chemora_grid_t grid, double* dev_fields, double* host_out, void* stream);

/* out[2q] = L2 = sqrt(h^3 sum c_q^2), out[2q+1] = Linf of the 7 constraints over the WHOLE
 * grid; nranks > 1: collective like chemora_norms (rank-ordered combination). */
int chemora_constraint_norms(chemora_grid_t grid, double* host_out, void* stream);
/* Combine rank-major per-rank partials (nranks x 14: [sum c_q^2, max|c_q|] x 7, from
 * chemora_constraints) in rank order into [L2, Linf] x 7. */
int chemora_constraint_norms_combine(const chemora_grid_desc* desc, const double* partials,
                                     int32_t nranks, double* out);

/* Model-driven tiling choice ("autotuning is model driven"): a
 * footprint/occupancy model prunes the stage-kernel tilings to <= 4 candidates, each is
 * timed on `trials` stage-1 launches (dt = 0: the state is not modified, the scratch set B
 * is), and the fastest is kept for this handle.  chosen[3] = {variant, band, #candidates};
 * ms_out (optional, >= 4 doubles) receives the best time per candidate (wave: per-step
 * estimate from stage 1-3 timings, or the two pair kernels; BSSN: stage 1).  Synchronises.
 * With nranks > 1 every rank must call it at the same point of its call sequence. */
int chemora_autotune(chemora_grid_t grid, int32_t trials, int32_t* chosen, double* ms_out,
                     void* stream);

/* ---- measurement */

/* Per-launch timing of the step (for roofline reporting): while enabled, every kernel launch
 * of chemora_rk4_step is bracketed by CUDA events recorded on the launching stream (up to
 * 4096 launches between reads).  chemora_read_launch_timing synchronises the stream and
 * returns, per launch slot s < 8 (wave temporally blocked path: 0 = stage pair 1+2, 1 =
 * stage pair 3+4; otherwise RK stage s+1), the summed milliseconds ms_sum[s] and the number
 * of launches counts[s] since the last read (both arrays of 8), then clears them.  Enabling
 * resets the record. */
int chemora_set_launch_timing(chemora_grid_t grid, int enable);
int chemora_read_launch_timing(chemora_grid_t grid, double* ms_sum, int32_t* counts, void* stream);

/* ---- testing hooks (not part of the user-facing contract) */

/* Select the kernel design of this handle.  WAVE: 0 = one thread per point,
 * 1 = same in plain order, 4 = persistent TMA z-march (every order; the default for order 8
 * when its 32x16 tiles fill the SMs; one kernel per RK stage), 8 = temporally blocked stage
 * pairs on 32x8 tiles with register-queue z stencils (orders 2, 4 and 6: the default there);
 * every wave design is bitwise identical.  BSSN: 0 =
 * two-phase SMEM table, 2 = fissioned G1/G2/G3, 3 = HBM derivative table + algebra kernels,
 * 4 = one fused kernel per stage with the derivatives on chip (SMEM plane tiles by TMA, TMEM
 * z-windows; default); results agree to rounding.  Refused after chemora_grid_connect_ipc. */
int chemora_set_kernel_variant(chemora_grid_t grid, int variant);

/* The kernel design chemora_rk4_step will run for this handle (the temporally blocked
 * variant 8 falls back to 0 where it does not apply: fd_order 8). */
int chemora_get_kernel_variant(chemora_grid_t grid, int* variant);

/* Copy state set `set` (0 = y, 1 = Q, 2 = B, 3 = C, in the current rotation) padded to host
 * [gf][Nz+2g][Ny+2g][Nx+2g].  Synchronises. */
int chemora_debug_get_set(chemora_grid_t grid, int set, double* host_dst, void* stream);

/* chemora_set_initial without the final halo exchange (ghosts left as cleared/copied). */
int chemora_set_initial_nofill(chemora_grid_t grid, int kind, const double* host_src,
                               const double* kind_params, uint64_t seed, void* stream);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* CHEMORA_H */
