/*
 * mm.h — C ABI of the B200 (sm_100a) ECSIM mass-matrix assembly library
 * (libmm.so).  arXiv 2604.19286, "Mass Matrix Assembly on Tensor Cores for
 * Implicit Particle-In-Cell Methods".
 *
 * What it computes (eq_mass_matrix_ecsim / eq_alpha_matrix /
 * eq_mass_matrix_general):
 *
 *   M^{ij}_{g g'} = sigma * sum_p s_p^{ij} W_pg W_pg'
 *   s_p^{ij} = q_p alpha_p^{ij}            (MM_TENSOR, 9 components)
 *            = q_p delta^{ij}              (MM_SCALAR, 1 component)
 *   alpha_p  = (I - C(omega_p) + omega_p omega_p^T) / (1 + |omega_p|^2),
 *   omega_p  = (qom * dt / 2) * B_p / c,   C(w) u = w x u
 *   W_pg     = prod_mu phi^(n)((x_p^mu - x_g^mu) / h^mu)     (eq_shape_bspline)
 *
 * with first-order (CIC, n = 1) or second-order (TSC, n = 2) B-splines, via
 * the paper's cell-local factorisation M = A B (eq_D_AB), particle batching
 * in K_t = 4 (eq_D_batches) and the support-group decomposition
 * (eq_group_partition), on FP64 DMMA tensor-core tiles.
 *
 * General conventions
 *   - No CUDA or torch types cross this boundary.  Every pointer argument
 *     documented as "device" is a CUDA device pointer on the current device;
 *     "host" pointers are ordinary host memory.  Streams are passed as
 *     `void*` holding a cudaStream_t (NULL = legacy default stream).
 *   - Every entry point returns an mm_status; on failure a thread-local
 *     message is available from mm_last_error().  No C++ exception crosses
 *     the ABI.  Argument checks are synchronous.
 *   - Grid geometry (readings R1, R2): node g sits at x = g*h,
 *     cell c = [c*h, (c+1)*h); cells = nodes per axis, periodic along axes
 *     1 and 2 always, and along axis 0 when the caller owns the whole axis
 *     (x_begin == 0 && x_end == n[0]).  Linearisation is row-major, axis 0
 *     slowest.
 *   - Output layout: out[(g*S + slot)*C + comp] with
 *       g    = ((ix - x_begin)*n[1] + iy)*n[2] + iz      (owned node rows)
 *       S    = (2n+1)^3 = 27 (order 1) | 125 (order 2)  stencil slots
 *       slot = ((dx+n)*(2n+1) + (dy+n))*(2n+1) + (dz+n), d = g' - g unwrapped
 *       comp = 3*i + j (MM_TENSOR) | 0 (MM_SCALAR)
 *     i.e. the full "27 neighbours x 9 components" (order 1) or
 *     "125 x 9" (order 2) node-stencil block per node.
 */
#ifndef MM_H_
#define MM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MM_OK = 0,
    MM_ERR_INVALID_ARG = 1,   /* bad pointer/size/enum/geometry                 */
    MM_ERR_DOMAIN = 2,        /* a particle lies outside the owned cell slab   */
    MM_ERR_NONFINITE = 3,     /* NaN/Inf in pos, q or B                        */
    MM_ERR_INCOMPATIBLE = 4,  /* handle/order/kind/precision mismatch          */
    MM_ERR_OUT_OF_MEMORY = 5, /* device allocation failed                      */
    MM_ERR_CUDA = 6,          /* CUDA runtime / launch error                   */
    MM_ERR_NCCL = 7           /* NCCL unavailable or a communicator call failed */
} mm_status;

typedef enum { MM_SCALAR = 1, MM_TENSOR = 9 } mm_kind; /* value = components C */

typedef enum {
    MM_FP64 = 0,   /* FP64 operands, FP64 DMMA 8x8x4 tiles (mma.sync), FP64 output        */
    MM_TF32 = 1,   /* TF32 operands (cvt.rna), FP32 accumulation in TMEM (tcgen05.mma
                      kind::tf32), FP32 output                                         */
    MM_TF32X3 = 2  /* split TF32 x = hi + lo, D += AhBh + AhBl + AlBh, FP32 output      */
} mm_precision;

typedef struct {
    int32_t n[3];    /* global cells = nodes per axis; n[a] >= 2*order+1        */
    double h[3];     /* spacing Delta x^mu > 0; domain [0, n*h)                  */
    int32_t x_begin; /* this rank owns cells/nodes ix in [x_begin, x_end)        */
    int32_t x_end;   /* single GPU: 0, n[0]  (x_end - x_begin >= order if slab)  */
} mm_grid;

typedef struct {
    double qom;   /* q_s/m_s             */
    double dt;    /* Delta t; beta_s = qom*dt/2             */
    double c;     /* speed of light, > 0 (normalised units: 1)   */
    double sigma; /* constant prefactor of eq_mass_matrix_general */
} mm_species;

typedef struct mm_sorted mm_sorted; /* opaque, library-owned device storage */
typedef struct mm_comm mm_comm;     /* opaque, library-owned NCCL communicator + comm stream */

typedef struct {
    int64_t np;        /* particles sorted                                        */
    int64_t np_padded; /* sorted slots incl. K-padding = seg_begin[nbins]         */
    int64_t nbins;     /* support-window bins (R12)                     */
    int64_t capacity;  /* allocated record slots (>= np + nbins*(k_pad-1))        */
    int32_t order;     /* 1 | 2                                                   */
    int32_t k_pad;     /* K tile the bins are padded to (multiple of 4)           */
    int32_t has_B;     /* 0: scalar-only handle (sorted without B)                */
    int32_t rec_stride; /* doubles per record: 8 (sorted with B) or 4 (without B)   */
    const int32_t *perm;      /* device [np_padded]: original index, -1 = pad     */
    const int32_t *seg_begin; /* device [nbins+1]: padded exclusive scan          */
    const int32_t *seg_count; /* device [nbins]: particles per bin                */
    const double *rec;        /* device [np_padded][rec_stride]: {xi_x,xi_y,xi_z,q,Bx,By,Bz,0}
                                 with B, {xi_x,xi_y,xi_z,q} for a scalar-only handle       */
} mm_sorted_info;

/*
 * mm_sort_by_cell — bin particles by their support window and pad the bins.
 *
 * PAPER.md:228 ("particles have been sorted by cell"), PAPER.md:242 (the last
 * batch of K_t particles is zero-padded) and PAPER.md:285-296
 * (eq_group_partition: particles grouped by identical support).  The bin of a
 * particle is its support-window base node j + b (b = 0 for CIC,
 * b_mu = -1 if xi_mu < 1/2 else 0 for TSC); axis 0 is
 * unwrapped and local: bx = c_x + b_x - x_begin + order - 1, nbins =
 * (x_end - x_begin + order - 1) * n1 * n2  (R12).  The sort is
 * STABLE (ties keep input order), so the permutation is unique and equals
 * the oracle's bit for bit.
 *
 *   g      host, grid/slab geometry
 *   order  1 | 2;  k_pad: multiple of 4 (4 or 8 typical)
 *   np     number of particles (0 allowed); must be < 2^31
 *   pos    device, [np][3] FP64 positions, row-major
 *   q      device, [np] FP64 charges
 *   B      device, [np][3] FP64 magnetic field at the particle, or NULL
 *          (scalar-only handle)
 *   stream cudaStream_t as void*
 *   inout  host, address of a handle pointer.  If *inout == NULL a new
 *          handle is created; otherwise the handle is reused (its device
 *          buffers grow if needed) and must have been created for the same
 *          grid and order.  On any error *inout is left unchanged.
 *
 * Ownership: the handle owns a sorted, padded copy of the particle data, so
 * the caller may free pos/q/B after the call.  Release with mm_free().
 * Pipeline: from MM_SORT_RECFIRST_MIN particles on (environment, read per call;
 * default 48e6, where the arrays exceed L2) the records are scattered first to
 * unstable slots and put in stable order per bin (one random pass instead of
 * three; the handle then holds an extra [capacity][8] FP64 scratch buffer).
 * Both pipelines give bit-identical results.
 * Synchronisation: the call enqueues its kernels on `stream` and then waits
 * for that stream once, to read back the error flags (MM_ERR_DOMAIN for a
 * particle whose cell is outside [x_begin,x_end) x [0,n1) x [0,n2) — never
 * clamped; MM_ERR_NONFINITE for NaN/Inf).
 */
mm_status mm_sort_by_cell(const mm_grid *g, int order, int k_pad, int64_t np, const double *pos,
                          const double *q, const double *B, void *stream, mm_sorted **inout);

/*
 * mm_sort_by_cell_mixed — the same sort for the production storage of PAPER.md:572
 * ("field values and particle positions are stored in FP32, while ... statistical
 * weights and the mass matrix use FP64"): pos and B are FP32 ([np][3] each, B may be
 * NULL), q is FP64.  Every value is widened exactly to FP64 before locate (R5), so the
 * result equals mm_sort_by_cell on the widened arrays bit for bit; the handle's records
 * are FP64 as always.  Arguments, ownership, errors and synchronisation as above.
 */
mm_status mm_sort_by_cell_mixed(const mm_grid *g, int order, int k_pad, int64_t np, const float *pos,
                                const double *q, const float *B, void *stream, mm_sorted **inout);

/*
 * mm_sort_by_cell_async — mm_sort_by_cell without its host round trip (a PIC step sorts and
 * assembles back to back on one stream: the host need not wait between them).  Same arguments
 * and device work; argument checks are synchronous as for mm_sort_by_cell.  The domain /
 * finiteness checks run on the device into a sticky status word that accumulates over every
 * sort of the handle until mm_sort_wait reports (and clears) it; np_padded is known only then.
 * A handle is returned (and created) even if the particles turn out to be invalid: the caller
 * must call mm_sort_wait before trusting any result computed from it, and frees it with mm_free.
 */
mm_status mm_sort_by_cell_async(const mm_grid *g, int order, int k_pad, int64_t np, const double *pos,
                                const double *q, const double *B, void *stream, mm_sorted **inout);

/*
 * mm_sort_wait — report the deferred status of the asynchronous sorts of a handle: waits for
 * `stream` (the sorts' stream, or one ordered after it), returns MM_ERR_DOMAIN /
 * MM_ERR_NONFINITE if any of them met an invalid particle since the last check (the handle is
 * then marked invalid), MM_OK otherwise; clears the sticky word.  MM_OK at once if nothing is
 * pending.  mm_sorted_view waits on the last asynchronous sort's stream by itself.
 */
mm_status mm_sort_wait(mm_sorted *h, void *stream);

/*
 * mm_resort_by_cell — incremental re-binning of the SAME particles after they moved (SURVEY.md
 * NEXT-1, the "sort & communicate" stage of a PIC cycle).  The handle must
 * hold a valid sort of np particles in the same order (same grid, order, k_pad; B given iff it
 * was).  Every particle is re-keyed; only those whose support-window bin changed update the bin
 * counters; each bin's new member list is its old stable slice minus the leavers plus its
 * arrivals, put back in ascending particle order; the records are rewritten from the new
 * positions.  The result (perm, seg_begin, records) is bit-identical to mm_sort_by_cell of the
 * new positions.  wait = 1: errors reported synchronously as by mm_sort_by_cell (the handle is
 * then invalid); wait = 0: deferred as by mm_sort_by_cell_async (mm_sort_wait).  Errors:
 * MM_ERR_INCOMPATIBLE (no valid previous sort, np or B presence differ), MM_ERR_DOMAIN,
 * MM_ERR_NONFINITE, MM_ERR_CUDA.
 */
mm_status mm_resort_by_cell(mm_sorted *h, int64_t np, const double *pos, const double *q, const double *B,
                            void *stream, int wait);

/* mm_sorted_view — read-only view of a handle's device arrays (see struct). */
mm_status mm_sorted_view(const mm_sorted *h, mm_sorted_info *out);

/*
 * mm_assemble — the mass matrix of one species from a sorted handle.
 *
 * Algorithm 1: for each support-window bin (= support
 * group), batches of K_t = 4 particles are contracted on FP64 DMMA 8x8x4 tiles
 * (eq_AB_batch, eq_mma_accumulate) and the finished block is scattered into the
 * node-stencil storage.  The operands are the per-axis pair
 * products of the B-spline weights (W_a W_b = q_x q_y q_z, eq_shape_bspline):
 * X = q_x q_y and Z = q_z s^{ij}, one product X Z^T per bin.
 *
 *   h          sorted handle (mm_sort_by_cell) for the same grid
 *   kind       MM_SCALAR | MM_TENSOR (MM_TENSOR needs a handle sorted with B)
 *   prec       MM_FP64 (DMMA, FP64 out) | MM_TF32 | MM_TF32X3 (tcgen05 kind::tf32,
 *              FP32 out; the TF32 variant "reported separately").
 * *   sp         host, species constants (qom, dt, c > 0, sigma)
 *   accumulate 0: out = M (the owned rows are overwritten);
 *              1: out += M (species sum)
 *   out        device, [(x_end-x_begin)*n1*n2][S][C] (layout above); FP64 for
 *              MM_FP64, FP32 for MM_TF32 / MM_TF32X3
 *   ghost      device, same element type, [mm_ghost_planes(order)][n1*n2][S][C], required
 *              when the grid is a slab (x_begin > 0 or x_end < n[0]) and
 *              ignored (may be NULL) otherwise.  Rows of nodes outside the
 *              slab are added here: order 1 -> plane 0 = node plane x_end;
 *              order 2 -> planes 0,1,2 = x_begin-1, x_end, x_end+1.  It is
 *              zeroed first unless accumulate = 1.
 *   stream     cudaStream_t as void*
 * Fully asynchronous.  The handle must not be re-sorted or freed until the
 * stream has passed this call.
 */
mm_status mm_assemble(const mm_sorted *h, mm_kind kind, mm_precision prec, const mm_species *sp,
                      int accumulate, void *out, void *ghost, void *stream);

/*
 * mm_deposit_moments — particle moments on the nodes with the assembly's machinery (SURVEY.md
 * NEXT-4; "any particle-to-grid scatter operation, where one MMA operand encodes
 * the deposited quantities and the other encodes the interpolation weights"):
 *   mom[g][m] = sigma * sum_p Q_p^m W_pg
 *   nq = 4:  Q_p = q_p (1, vx, vy, vz)                                    (charge, current)
 *   nq = 10: Q_p = q_p (1, vx, vy, vz, vx vx, vx vy, vx vz, vy vy, vy vz, vz vz)   (implicit
 *            moment method quantities; second moments upper triangle row-major)
 * per support-window bin on FP64 DMMA tiles (A = node weights, B = quantities).
 *   h      sorted handle (with or without B); the particles are those given to the sort
 *   sp     host; only sigma is used
 *   v      device, [np][3] FP64 velocities in the caller's particle order (the order given to
 *          mm_sort_by_cell; read through the handle's permutation)
 *   accumulate 0: out = mom; 1: out += mom
 *   out    device, FP64 [(x_end-x_begin)*n1*n2][nq] (node rows as in mm_assemble)
 *   ghost  device, FP64 [mm_ghost_planes(order)*n1*n2][nq] for slab grids (zeroed unless
 *          accumulate), NULL for the whole domain; reduced like the mass matrix's ghost planes
 * Asynchronous.
 */
mm_status mm_deposit_moments(const mm_sorted *h, int nq, const mm_species *sp, const double *v, int accumulate,
                             double *out, double *ghost, void *stream);

/*
 * mm_gather_field — a nodal vector field interpolated to the sorted particles with the same
 * B-spline weights ("B(x_p) ... the magnetic field interpolated to the particle
 * position"):  F_p = sum_g W_pg F_g.  The result REPLACES the B fields of the handle's records,
 * so a following mm_assemble uses it (gather -> alpha -> mass matrix, no re-sort), and, if Fp is
 * not NULL, is also written in the caller's particle order.
 *   h      handle sorted WITH B (MM_ERR_INCOMPATIBLE otherwise); modified in place
 *   F      device, FP64 [n0*n1*n2][3], the field at every node of the whole periodic domain
 *          (also for a slab handle: the window of a bin may reach one plane beyond the slab)
 *   Fp     device, FP64 [np][3] in the order given to mm_sort_by_cell, or NULL
 * Asynchronous.
 */
mm_status mm_gather_field(mm_sorted *h, const double *F, double *Fp, void *stream);

/*
 * mm_apply — y (+)= M E: the matrix-free product of an assembled FP64 mass
 * matrix with a nodal field, the operation the implicit field solve performs
 * with it ((L + sum_s M_s) E = b, eq_field_eq):
 *   y[g][i] = sum_slot sum_j M[g][slot][3i+j] E[wrap(g + d(slot))][j]   (MM_TENSOR)
 *   y[g]    = sum_slot M[g][slot] E[wrap(g + d(slot))]                  (MM_SCALAR)
 *   g          host, grid; whole periodic domain only (x_begin = 0, x_end = n[0]),
 *              else MM_ERR_INCOMPATIBLE
 *   M          device, FP64 [n0*n1*n2][S][C] (mm_assemble's layout)
 *   E, y       device, FP64 [n0*n1*n2][3] (MM_TENSOR) or [n0*n1*n2] (MM_SCALAR);
 *              y must not alias E or M
 *   accumulate 0: y = M E; 1: y += M E
 * Asynchronous on `stream`.
 */
mm_status mm_apply(const mm_grid *g, int order, mm_kind kind, const double *M, const double *E, double *y,
                   int accumulate, void *stream);

/*
 * mm_slab_partition — particle migration between x-slabs, the first half of the "sort &
 * communicate" stage: a STABLE 3-way partition of a
 * rank's particles by the slab of their cell along x (cell = floor(x/h), IEEE quotient, R5):
 *   class 0: stays      (cell in [x_begin, x_end))
 *   class 1: to r - 1   (leaves through x_begin)
 *   class 2: to r + 1   (leaves through x_end)
 * The cells outside the slab are split half-and-half between the two directions (periodic):
 * a leaver goes towards the nearer side of the ring.  A particle that moved further than the
 * neighbouring slab is forwarded again by the neighbour (multi-hop: the caller repeats
 * partition + exchange on the received particles until no rank has leavers, e.g.
 * paper_2604_19286_b200.slab.migrate).  Non-finite or out-of-domain positions are kept in
 * class 0 (mm_sort_by_cell reports them).
 *   g          host, grid with this rank's slab
 *   pos,q,B    device, FP64 [np][3], [np], [np][3] (B may be NULL)
 *   pos_out,q_out,B_out  device, same shapes: [class 0 | class 1 | class 2], input order kept
 *              inside every class; must not alias the inputs
 *   counts     host int64[3]: particles per class
 * Synchronous (waits for `stream` to read the counts back).
 */
mm_status mm_slab_partition(const mm_grid *g, int64_t np, const double *pos, const double *q, const double *B,
                            double *pos_out, double *q_out, double *B_out, int64_t counts[3], void *stream);

/*
 * mm_ghost_add — add `nplanes` received ghost node planes into owned rows (FP64 output)
 * (the reduction step of the slab decomposition):
 *   out[((first_plane + k)*n1*n2 + r)*S*C + e] += recv[(k*n1*n2 + r)*S*C + e]
 * for k < nplanes.  `first_plane` is relative to x_begin.  Asynchronous.
 */
mm_status mm_ghost_add(const mm_grid *g, int order, mm_kind kind, double *out, const double *recv,
                       int first_plane, int nplanes, void *stream);

/*
 * Multi-GPU: x-slab decomposition with particles owned by cell and the ghost-plane reduction over
 * NCCL send/recv (north_star, the "sort & communicate"
 * stage and the task-based overlap of communication with compute).  One process per GPU.
 *
 * mm_comm_unique_id — ncclGetUniqueId into `uid` (host, 128 bytes).  Call on one rank and
 *   broadcast the bytes to all ranks (e.g. over a torch.distributed process group).
 * mm_comm_create — ncclCommInitRank(nranks, uid, rank) on the CURRENT device, plus a
 *   non-blocking communication stream owned by the communicator.  Collective over the ranks.
 *   Released only by mm_comm_free (which waits for the comm stream).
 * NCCL is loaded at run time (libnccl.so.2); without it these calls return MM_ERR_NCCL.
 */
mm_status mm_comm_unique_id(void *uid);
mm_status mm_comm_create(int nranks, int rank, const void *uid, mm_comm **out);
void mm_comm_free(mm_comm *comm);

/*
 * mm_ghost_exchange — the ghost-plane reduction of one rank's slab on a periodic ring of ranks:
 *   order 1: ghost plane 0 (node plane x_end)     -> rank r+1, added into its owned plane 0
 *   order 2: ghost plane 0 (node plane x_begin-1) -> rank r-1, added into its last owned plane;
 *            ghost planes 1, 2 (x_end, x_end+1)   -> rank r+1, added into its owned planes 0, 1
 * Every rank posts send(next), recv(prev), send(prev), recv(next) in one NCCL group on the
 * communicator's stream, which first waits for `stream`; `stream` waits for the transfer before
 * the add kernels.  Asynchronous.  Collective: every rank of the communicator calls it.
 *   comm    communicator of nranks ranks; rank r owns the slab `g` (slab width >= order on
 *           every rank).  A communicator of ONE rank exchanges with itself (self ring): then `g`
 *           must be the whole domain and the ghost planes are those of the slab [0, n0).
 *   g, order, kind, prec  as for mm_assemble; prec selects FP64 (out/ghost double) or FP32
 *   out     device, owned rows [(x_end-x_begin)*n1*n2][S][C] (receives the neighbours' planes)
 *   ghost   device, this rank's ghost planes [mm_ghost_planes(order)*n1*n2][S][C] (sent; not
 *           modified)
 * Receive buffers are owned by the communicator; successive exchanges on one communicator must
 * be ordered on one stream.  Errors: MM_ERR_INCOMPATIBLE for a whole grid with > 1 rank or a
 * slab grid with 1 rank; MM_ERR_NCCL for a failed NCCL call.
 */
mm_status mm_ghost_exchange(mm_comm *comm, const mm_grid *g, int order, mm_kind kind, mm_precision prec, void *out,
                            void *ghost, void *stream);

/*
 * mm_assemble_slab — mm_assemble on this rank's slab followed by the ghost reduction, with the
 * exchange overlapped with the assembly: the bin planes whose support windows
 * reach a ghost plane (order 1: the last bin plane; order 2: the first and the last two) are
 * assembled first into `ghost`, the ghost planes travel on the communicator's stream while the
 * interior bins are assembled on `stream`, then the received planes are added into `out`.  On
 * return (stream order) `out` holds the complete owned rows of the global mass matrix.
 *   h, kind, prec, sp   as for mm_assemble (h sorted for this rank's slab grid; with a one-rank
 *                       communicator, for the whole grid: the self ring)
 *   accumulate          0: out = M; 1: out += M (species sum)
 *   out                 device, owned rows (layout of mm_assemble)
 *   ghost               device scratch [mm_ghost_planes(order)*n1*n2][S][C]; zeroed by the call
 *   comm, stream        communicator of this rank; cudaStream_t as void*
 * Asynchronous; collective over the communicator.  Errors as mm_assemble and mm_ghost_exchange.
 */
mm_status mm_assemble_slab(const mm_sorted *h, mm_kind kind, mm_precision prec, const mm_species *sp, int accumulate,
                           void *out, void *ghost, mm_comm *comm, void *stream);

/* Number of ghost node planes of a slab: 1 (order 1) or 3 (order 2). */
int mm_ghost_planes(int order);

/* Elements (doubles) of the owned output: (x_end-x_begin)*n1*n2*S*C, or -1. */
int64_t mm_out_elems(const mm_grid *g, int order, mm_kind kind);

/* Release a handle (NULL is a no-op).  Synchronises the device first. */
void mm_free(mm_sorted *h);

/* Thread-local description of the last failure of this thread (host string). */
const char *mm_last_error(void);

/* Library version string, e.g. "mm-b200 0.1 sm_100a". */
const char *mm_version(void);

/* Number of kernel launches this library has issued since load (host counter,
 * used by the benchmark's gpu_launches claim). */
int64_t mm_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* MM_H_ */
