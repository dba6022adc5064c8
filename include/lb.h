/*
 * lb.h -- C ABI of the B200-native D3Q19 binary-fluid lattice-Boltzmann step.
 *
 * What one step computes (sec. 2.1.1; readings R1-R22 of
 * DESIGN.md, which spell out the equations the paper only names):
 *   1. moments rho = sum_i f_i, j = sum_i c_i f_i, phi = sum_i g_i            (A.3)
 *   2. "Order Parameter Gradients": central grad phi, 7-point lap phi        (A.2)
 *   3. chemical potential mu and "Chemical Stress" P_ab                       (A.4)
 *   4. force F = -div P ("the divergence of the 'Chemical stress'")           (A.5)
 *   5. "Collision": BGK of f with Guo forcing, BGK of g towards g^eq(phi,u,Gamma mu)
 *                                                                             (A.6-A.7)
 *   6. "Propagation": "displacing the fluid data one lattice spacing in the
 *      appropriate direction", periodic                                       (A.8)
 *   7. halo exchange between z-slabs ("each local sub-domain is surrounded by a
 *      halo region populated using neighboring sub-domain data")
 *
 * Conventions
 *   - All field values are IEEE fp64 ("a set of double precision values
 *     at each lattice point").
 *   - Canonical D3Q19 order: rest first, then the 18 moving velocities in
 *     descending lexicographic (cx, cy, cz) (reading R1).
 *   - Site index s = x + nx*(y + ny*z), x fastest.  A distribution array is
 *     f[p*nloc + s], p = 0..18, nloc = nx*ny*nz_local.
 *   - State = the PRE-collision (post-propagation) f and g at integer time t (R12).
 *
 * Ownership: the caller owns every host array and the library never keeps a
 * pointer to one after a call returns; the library owns all device memory, its
 * CUDA stream and (for lb_create_slab) its NCCL communicator.  Host<->device
 * copies are synchronous: on return the data has been transferred.  Host
 * arrays may be pageable or page-locked (page-locked is faster).
 *
 * Errors: every int-returning call returns LB_OK (0) or a negative code; the
 * handle's lb_last_error() then holds a one-line message.  After LB_ECUDA or
 * LB_ENCCL the handle is unusable except for lb_destroy / lb_last_error.
 * A handle is thread-compatible: one thread at a time.
 */
#ifndef LB_H
#define LB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  LB_OK = 0,
  LB_EINVAL = -1,   /* null pointer, bad extent, bad parameter, nsteps < 0 ...     */
  LB_ENOMEM = -2,   /* device or host allocation failed                            */
  LB_ECUDA = -3,    /* CUDA runtime failure; handle unusable                       */
  LB_ENCCL = -4,    /* NCCL failure; handle unusable                               */
  LB_ESTATE = -5,   /* step / get before any set_state or init_equilibrium        */
  LB_ENUMERIC = -6  /* some site had rho <= 0 or a non-finite value (R22)  */
};

/* Physical parameters of the problem statement (BASELINE north_star; R2, R10).
 * Free energy  F[phi] = sum_x A/2 phi^2 + B/4 phi^4 + kappa/2 |grad phi|^2.    */
typedef struct {
  double tau_f;    /* BGK relaxation time of f, finite and > 1/2                  */
  double tau_g;    /* BGK relaxation time of g, finite and > 1/2                  */
  double A, B;     /* bulk free-energy coefficients, finite                        */
  double kappa;    /* interfacial coefficient, finite and >= 0                     */
  double mobility; /* M >= 0; internally Gamma = M / (tau_g - 1/2)   (R10)         */
} lb_params;

typedef struct lb_ctx lb_t;

/* Library version string (static storage). */
const char* lb_version(void);

/* Whole periodic lattice nx x ny x nz on the current CUDA device.
 * Extents must be >= 3.  *out receives the handle (NULL on failure). */
int lb_create(int nx, int ny, int nz, const lb_params* params, lb_t** out);

/* Same lattice, decomposed inside this handle into nslabs z-slabs of nz/nslabs
 * planes each, whose halos are exchanged by device-to-device copies on this
 * GPU ("loopback" transport).  Results are bitwise identical to lb_create; it
 * exists to exercise the slab index maps on one GPU.  nz % nslabs == 0 and
 * nz/nslabs >= 2.  The host arrays of set/get are still the whole lattice. */
int lb_create_loopback(int nx, int ny, int nz, const lb_params* params, int nslabs, lb_t** out);

/* Bootstrap for lb_create_slab: rank 0 fills 128 bytes (an ncclUniqueId); the
 * caller broadcasts them to all ranks by any means.  */
int lb_nccl_get_unique_id(void* id128);

/* Rank `rank` of a z-slab decomposition over `nranks` processes, one GPU each
 * (the current CUDA device).  Rank r owns global z in [r*L, (r+1)*L), L =
 * nz/nranks >= 2; halos travel by NCCL send/recv to ranks r+-1 (mod nranks).
 * Collective: every rank must call it.  Host arrays of set/get/init are this
 * rank's slab only (nloc = nx*ny*L sites).  nranks == 1 is lb_create. */
int lb_create_slab(int nx, int ny, int nz, const lb_params* params, int nranks, int rank,
                   const void* id128, lb_t** out);

/* Number of sites this handle's host arrays hold (nloc).  Returns 0 for NULL. */
size_t lb_local_sites(const lb_t* h);

/* One rank of a z-slab decomposition, bootstrapped by the caller instead of NCCL
 * (collective over all ranks, like lb_create_slab).  allgather(ctx, send, recv,
 * bytes) must gather `bytes` host bytes from every rank into recv (nranks * bytes,
 * rank order) and return 0; it is called during this call, by lb_init_equilibrium
 * and by lb_step on propagation-only steps, until lb_destroy (the library keeps
 * fn and ctx).  The halo transport is the peer one (CUDA IPC mappings of the
 * neighbours' buffers, device-side ordering): if the neighbours' memory cannot be
 * mapped, LB_ENCCL.  Ranks may share a GPU here (tests), since nothing of this
 * path needs one communicator rank per device. */
typedef int (*lb_allgather_fn)(void* ctx, const void* send, void* recv, size_t bytes);
int lb_create_slab_ext(int nx, int ny, int nz, const lb_params* params, int nranks, int rank,
                       lb_allgather_fn allgather, void* ctx, lb_t** out);

/* Load the state: f, g are host arrays of 19*nloc doubles each, canonical
 * layout.  Bitwise: lb_get_state right after returns exactly these bits. */
int lb_set_state(lb_t* h, const double* f, const double* g);

/* Initialise at local equilibrium from macroscopic host fields (R15):
 * f = f^eq(rho, u), g = g^eq(phi, u, Gamma*mu[phi]) with mu from the 7-point
 * Laplacian of phi (A.4).  rho: nloc doubles or NULL (rho = 1); u: 3*nloc
 * doubles u[a*nloc + s] or NULL (u = 0); phi: nloc doubles (required).
 * Collective for slabs (exchanges phi halo planes). */
int lb_init_equilibrium(lb_t* h, const double* rho, const double* u, const double* phi);

/* Advance nsteps >= 0 timesteps; returns after the device has finished.
 * LB_ENUMERIC if any site had rho <= 0 or a non-finite f/g/phi during these
 * steps (R22): the kernels record the first offending (step, site)
 * and lb_last_error names it -- global (x, y, z) and the step within this call;
 * the flag is read once, at the end, so the state has advanced all nsteps.
 * Collective for slabs. */
int lb_step(lb_t* h, int nsteps);

/* Optional: capture the CUDA graphs lb_step replays (8 steps each, one per
 * buffer parity) now instead of at the first lb_step that can use them.  No
 * device work and no change of state; a no-op where graphs are not used (ranks,
 * per-launch profiling, LB_TUNE_GRAPHS 0).  Lets a caller keep graph capture out
 * of a timed region (bench.py). */
int lb_prepare(lb_t* h);

/* Read the state back into host arrays of 19*nloc doubles each. */
int lb_get_state(lb_t* h, double* f, double* g);

/* Order parameter phi = sum_i g_i of the current state, nloc doubles. */
int lb_get_phi(lb_t* h, double* phi);

/* Frees device memory, the stream and the communicator.  NULL-safe. */
void lb_destroy(lb_t* h);

/* Last error message of this handle ("" if none); for a NULL handle, the last
 * error of a failed lb_create* call in this thread.  Owned by the library. */
const char* lb_last_error(const lb_t* h);

/* ---- measurement support (bench.py) ------------------------------------ */

/* The cudaStream_t every kernel and copy of this handle is issued on. */
void* lb_stream(const lb_t* h);

/* Kernels launched by this handle since creation (host-side count). */
long long lb_launch_count(const lb_t* h);

/* Per-kernel CUDA-event timing.  When enabled, every launch is bracketed by
 * events on the handle's stream; totals accumulate until reset. */
int lb_profile_enable(lb_t* h, int on);
int lb_profile_reset(lb_t* h);
/* Entry i (0 <= i < lb_profile_count): kernel name (static storage), summed
 * device milliseconds and number of timed launches. */
int lb_profile_count(const lb_t* h);
int lb_profile_entry(const lb_t* h, int i, const char** name, double* total_ms, long long* launches);

/* Algorithmic HBM bytes one site update moves in the step kernel (reads and
 * writes of f and g once each: 38 * 2 * 8 = 608).  Used for the roofline. */
double lb_bytes_per_site(void);

/* ---- test support ------------------------------------------------------- */

/* Integer propagation map of A.8 as the device code implements it: the
 * composition of the kernels' push addressing with the halo plan of an
 * nslabs-way z-slab decomposition, inverted into a pull map over the GLOBAL
 * lattice:  out[p*N + s] = canonical global index of the site whose
 * post-collision component p streams into site s (N = nx*ny*nz, int64).
 * Host-only; no GPU needed.  LB_EINVAL on bad sizes or if the composition is
 * not a permutation. */
int lb_debug_propagation_map(int nx, int ny, int nz, int nslabs, int64_t* out);

/* Propagation only (collision = identity) for nsteps steps on the device, with
 * the same kernel addressing and halo exchanges as lb_step.  Test support. */
int lb_debug_stream(lb_t* h, int nsteps);

/* Launch knobs of the step kernels, for measurement (the defaults are the tuned
 * choice; nothing reads the environment).  Results are bitwise the same for any
 * value.  Keys:
 *   LB_TUNE_ZCHUNK    planes per z-chunk of a CTA (0: automatic, step_zchunk)
 *   LB_TUNE_VARIANT   a kernel alternative kept for A/B measurement: 1 = the
 *                     Cahn-Hilliard warp-specialised kernel with a 5-plane phi
 *                     ring (phi issued 3 planes ahead instead of 4); 0 the default
 *   LB_TUNE_TILE_ROWS tile rows of the binary-fluid and Cahn-Hilliard step kernels,
 *                     4 or 8 (0: automatic); resets the z-chunk to its automatic value
 *   LB_TUNE_BAND_ROWS block order: tiles walked in bands of this many tile rows,
 *                     column by column (1: row-major, the default)
 *   LB_TUNE_RESID     CTAs assumed resident at a time by the block order (0: the
 *                     kernel's occupancy on this device)
 *   LB_TUNE_GRAPHS    0: step without CUDA graphs; 1 (default): graphs of 8 steps
 *   LB_TUNE_L2_BOX, LB_TUNE_L2_FTILE, LB_TUNE_L2_GTILE
 *                     L2 eviction policy of the warp-specialised kernel's copies of
 *                     the g halo box, the f tile and the g tile: 0 evict_normal,
 *                     1 evict_first, 2 evict_last, 3 evict_unchanged
 * LB_EINVAL for an unknown key or a value out of range. */
enum {
  LB_TUNE_ZCHUNK = 1,
  LB_TUNE_BAND_ROWS = 2,
  LB_TUNE_RESID = 3,
  LB_TUNE_GRAPHS = 4,
  LB_TUNE_L2_BOX = 5,
  LB_TUNE_L2_FTILE = 6,
  LB_TUNE_L2_GTILE = 7,
  LB_TUNE_TILE_ROWS = 8,
  LB_TUNE_VARIANT = 9
};
int lb_debug_tune(lb_t* h, int key, int value);

/* ---- NEXT-2 variant: finite-difference Cahn-Hilliard (R29-R33) ----
 * A handle whose state is (f, phi): phi is a field updated each step by
 *   phi <- phi - sum_a [J_a(x + e_a/2) - J_a(x - e_a/2)] + M lap mu,
 *   J = u_f * phi_upwind, u_f = (u(x) + u(x + e_a))/2, u = j/rho   (R30, R31)
 * instead of the g distribution, and f collides with the chemical stress in
 * its equilibrium and a three-rate MRT (model 1 of lb_set_collision, R32).
 * A periodic lattice on the current GPU (or z-slabs, below); nx even, else LB_EINVAL;
 * tau_f and tau_g of params are unused, M enters the update directly.
 * lb_step, lb_get_phi, lb_init_equilibrium (f = f^eq(rho, u) of R8, phi as
 * given), lb_destroy work as for other handles; lb_set_state / lb_get_state
 * return LB_EINVAL (use the _ch pair: f canonical 19*nloc doubles, phi nloc). */
int lb_create_ch(int nx, int ny, int nz, const lb_params* params, double tau_shear, double tau_bulk,
                 double tau_ghost, lb_t** out);
/* The same variant on z-slabs (nz % slabs == 0, nz/slabs >= 2), in one handle on this
 * GPU (loopback; host arrays = the whole lattice) or one rank per GPU (collective;
 * host arrays = this rank's slab).  Before each step the f planes z_lo / z_hi (all
 * 19 components: u = j/rho at z +- 1) go to the neighbours' ghost planes and phi
 * two planes each way; after it, the f components that left the slab.  Bitwise
 * equal to lb_create_ch. */
int lb_create_ch_loopback(int nx, int ny, int nz, const lb_params* params, double tau_shear, double tau_bulk,
                          double tau_ghost, int nslabs, lb_t** out);
int lb_create_ch_slab(int nx, int ny, int nz, const lb_params* params, double tau_shear, double tau_bulk,
                      double tau_ghost, int nranks, int rank, const void* id128, lb_t** out);
int lb_set_state_ch(lb_t* h, const double* f, const double* phi);
int lb_get_state_ch(lb_t* h, double* f, double* phi);

/* ---- NEXT-4 workload: the paper's liquid crystal (R34-R45) ----------
 * "an 'order parameter' field (a 3x3 tensor, which is symmetric and traceless)"
 * evolved by "a finite difference implementation of the Beris-Edwards model with
 * the Landau-de Gennes free energy functional" ("LC Update") and its "Advection",
 * coupled to the LB fluid by "the divergence of the 'Chemical stress'"
 * (PAPER.md P:158-183).  Per step (R43): grad Q and lap Q (R37); molecular field
 *   H = -A0 (1 - gamma/3) Q + A0 gamma (Q Q - I Q:Q/3) - A0 gamma (Q:Q) Q + kappa lap Q;
 * stress sigma (R38, Beris-Edwards, p0 = -f); F = div sigma (R39); Guo BGK of f
 * with tau_f (R40), whose u' = (j + F/2)/rho becomes the stored velocity; LC update
 *   Q <- Q - div J + S(W, Q) + Gamma H   (R41, R42: upwind J, W = grad u, stored u);
 * propagation of f.  State (R34): f canonical (19*nloc), Q by its five components
 * (xx, xy, xz, yy, yz) as q[c*nloc + s], and the stored velocity u[a*nloc + s].
 * A periodic lattice on the current GPU (or z-slabs, below); nx even, else LB_EINVAL.  lb_step,
 * lb_destroy, lb_last_error, lb_stream and the profiling calls work as for other
 * handles; lb_set_state, lb_get_state, lb_init_equilibrium, lb_get_phi and
 * lb_set_collision return LB_EINVAL. */
typedef struct {
  double tau_f;  /* BGK relaxation time of f, finite and > 1/2                     */
  double A0;     /* Landau-de Gennes bulk constant, finite                          */
  double gamma;  /* Landau-de Gennes "temperature" parameter, finite                */
  double kappa;  /* elastic constant, finite and >= 0                               */
  double xi;     /* flow-aligning parameter, finite                                 */
  double Gamma;  /* rotational diffusion constant, finite and >= 0                  */
} lb_lc_params;

int lb_create_lc(int nx, int ny, int nz, const lb_lc_params* params, lb_t** out);
/* The same workload decomposed into z-slabs (nz % slabs == 0, nz/slabs >= 2): inside
 * one handle on this GPU (loopback; host arrays = the whole lattice), or one rank
 * per GPU (collective like lb_create_slab; host arrays = this rank's slab).  Before
 * each step the Q planes z_lo, z_lo+1 / z_hi-1, z_hi and the u planes z_lo / z_hi go
 * to the neighbours' ghost planes; after it, the f components that left the slab
 * (device copies, or NCCL send/recv between ranks).  Bitwise equal to lb_create_lc. */
int lb_create_lc_loopback(int nx, int ny, int nz, const lb_lc_params* params, int nslabs, lb_t** out);
int lb_create_lc_slab(int nx, int ny, int nz, const lb_lc_params* params, int nranks, int rank, const void* id128,
                      lb_t** out);
/* Host arrays: f 19*nloc, q 5*nloc, u 3*nloc doubles (canonical layouts above);
 * set/get round trip bitwise. */
int lb_set_state_lc(lb_t* h, const double* f, const double* q, const double* u);
int lb_get_state_lc(lb_t* h, double* f, double* q, double* u);
/* R45 initial state from host fields: f = f^eq(rho, u) (R8), Q = S0 (n n - I/3) with
 * S0 = 1/4 + 3/4 sqrt(1 - 8/(3 gamma)) (needs gamma > 8/3, else LB_EINVAL), stored
 * velocity = u.  rho: nloc doubles or NULL (1); u: 3*nloc or NULL (0); n: unit
 * directors, 3*nloc doubles n[a*nloc + s] (required). */
int lb_init_lc(lb_t* h, const double* rho, const double* u, const double* n);

/* Collision model of f (readings R23-R27).
 *   model 0 (default, the paper path): BGK of f with tau_f of lb_params and the
 *     Guo force F = -div P (R5, R7); the tau arguments are ignored.
 *   model 1: the chemical stress P in the second moment of f's equilibrium
 *     (no force, u = j/rho) and a three-rate MRT of f: the traceless stress
 *     relaxes with tau_shear (viscosity (tau_shear - 1/2)/3), its trace with
 *     tau_bulk, the ghost modes with tau_ghost; tau_f of lb_params is unused.
 *     g is unchanged (BGK with tau_g, R9/R10), with the force-free u.
 * Each tau finite and > 1/2, else LB_EINVAL.  Takes effect at the next lb_step. */
int lb_set_collision(lb_t* h, int model, double tau_shear, double tau_bulk, double tau_ghost);

/* Which step kernel lb_step uses: 0 = default (the warp-specialised kernel for
 * even nx, with the phi exchange of kernel 3 where the step's blocks -- 32 x 8
 * tiles x z-chunks -- fit in one wave on the SMs, e.g. 64^3 and 128^3; else the
 * tile kernel), 1 = the tile kernel (halo box per CTA), 2 = the warp-specialised
 * tile kernel (stencil and collision on separate warps; needs nx even, else
 * LB_EINVAL), 3 = the warp-specialised kernel with the phi exchange (the stencil
 * loads the g tile only and takes the phi halo from the neighbouring tiles' CTAs
 * through an L2-resident phi array whose unwritten sites hold a sentinel NaN,
 * summing it from g where the owner runs behind; one periodic slab, nx % 32 == 0,
 * ny % 8 == 0, else LB_EINVAL; allocates two nx*ny*nz phi arrays).  All give
 * bitwise identical results.  Test / measurement support. */
int lb_debug_step_kernel(lb_t* h, int which);

/* Halo transport of a slab handle.  mode -1: returns the current mode (0 or 1);
 * 0: exchange -- kernels push into ghost planes, then device copies (loopback) or
 *    NCCL send/recv (ranks) move them, and the phi ghost planes likewise;
 * 1: peer (fused) -- the step kernel stores the components leaving the slab
 *    directly into the neighbour's next-state buffer, and K_phi its edge planes
 *    into the neighbour's phi ghost planes (same GPU for loopback; NVLink P2P
 *    through CUDA IPC mappings between ranks); only a one-double NCCL send/recv
 *    per phase orders the ranks.
 * Default: 1 for loopback and for ranks whose neighbours' memory could be mapped
 * (checked end to end at lb_create_slab), else 0.  Both give bitwise identical
 * results.  LB_EINVAL for a single
 * periodic slab or a rank handle without peer mappings. */
int lb_debug_halo_mode(lb_t* h, int mode);

/* One step in three host-visible phases (test support; peer transport of a slab
 * handle of the binary fluid): phase 0 = K_phi of the slab edges into the
 * neighbours' ghost planes, phase 1 = the step kernel, its pushes into the
 * neighbours and the end-of-step role swap, phase 2 = the lb_step epilogue (wait
 * for the neighbours' pushes, numerical-domain and timeout report).  Each phase
 * returns after the device has finished it, so ranks that put a barrier between
 * phases never have a kernel waiting on another rank's: the device-side waits of
 * the next phase are already satisfied.  LB_EINVAL for other handles. */
int lb_debug_step_phase(lb_t* h, int phase);

/* lb_debug_propagation_map for the peer transport: the destinations come from the
 * kernels' own address arithmetic with the neighbouring slabs' buffers (no ghost
 * planes, no halo plan).  Must equal lb_debug_propagation_map.  Host-only. */
int lb_debug_propagation_map_peers(int nx, int ny, int nz, int nslabs, int64_t* out);

/* Memory-safety check (test support; this pool has no compute-sanitizer): every
 * field buffer (f/g A and B, phi, Q, u, the phi-exchange arrays) is allocated with
 * 64 KB guard zones on both sides holding a fixed byte pattern.  Returns the
 * number of guard bytes that no longer hold it -- 0 unless some kernel or copy
 * stored outside its buffer -- or a negative LB_* code. */
long long lb_debug_guards(lb_t* h);

/* Built with -DLB_CHECKED (liblb_checked.so, _build.build(checked=True))?  1 or 0.
 * In that build the kernels check their computed indices (wrapped halo boxes,
 * ghost phi planes, exchange sites, push targets); lb_debug_check returns the
 * source line (in the kernel files) of the first check that failed, 0 if none,
 * or a negative LB_* code.  Always 0 in the product build. */
int lb_debug_checked(void);
int lb_debug_check(lb_t* h);

/* Block order of the step kernels (host-only): for block L of a launch over ntx x
 * nty tiles and nch z-chunks, out[3L .. 3L+2] = (tile column, tile row, chunk) as
 * the kernels compute it with `resid` CTAs resident and bands of `band` tile rows
 * (LB_TUNE_BAND_ROWS); band < 0: bands of -band rows in the order of a z-slab
 * with the peer transport, whose edge chunks (first and last) run after the
 * interior ones when there are >= 3.  Every (tile, chunk) appears exactly once.
 * out holds 3 * ntx * nty * nch ints.  LB_EINVAL on bad arguments. */
int lb_debug_tile_order(int ntx, int nty, int nch, int resid, int band, int* out);

/* Halo plan of a slab decomposition (host-only; no GPU needed): for rank r of
 * nranks, the ranks it sends its +z and -z halo to, and the number of doubles
 * per message: distributions (10 components x nx*ny) and phi (2 planes x nx*ny).
 * out[0]=up, out[1]=down, out[2]=dist doubles, out[3]=phi doubles. */
int lb_halo_plan(int nx, int ny, int nz, int nranks, int rank, int64_t out[4]);

#ifdef __cplusplus
}
#endif
#endif /* LB_H */
