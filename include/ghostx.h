/*
 * ghostx.h — C ABI of the B200-native ghost-cell exchange library
 * (libghostx.so, built from paper_2403_12179_b200/csrc/).
 *
 * It replaces the hot path of the reference package miniamr_core
 * (/root/reference/pkg/src/miniamr_core/comm.py):
 *
 *   plan builder   _shift_candidates / _build_copy_segments / CommPlan /
 *                  plan_build_fill_boundary / parallel_copy plan part
 *                  (comm.py:250-309, :413-424)        -> ghx_plan_build_*
 *   executor       _execute_plan (local fused copy, pack, Bus send/recv,
 *                  unpack; comm.py:316-380)            -> ghx_exec_*
 *   BoxArray ctor  O(n^2) disjointness check (mesh.py:203-205)
 *                                                       -> ghx_boxes_disjoint
 *
 * Conventions (all plain C types, no torch types):
 *  - a box is six int64: lo0 lo1 lo2 hi0 hi1 hi2, padded to 3 axes with
 *    lo = hi = 0 on unused axes (core/mesh.py:31-40);
 *  - fab storage is F-order (nx, ny, nz, ncomp) over the fab's storage
 *    (grown) box, element size 4 or 8 bytes, copied as raw words;
 *  - every function returns GHX_OK (0) or a GHX_E* code and never throws;
 *    ghx_last_error() returns a thread-local message for the last failure;
 *  - plans are immutable after build and may be shared by threads; an exec
 *    handle is owned by one rank (thread or process) at a time;
 *  - device calls are stream-ordered on the cudaStream_t passed as void*.
 */
#ifndef GHOSTX_H
#define GHOSTX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GHX_OK 0
#define GHX_EINVAL 1
#define GHX_ECUDA 2
#define GHX_ENOMEM 3
#define GHX_EOVERLAP 4

#define GHX_MODE_FILL_BOUNDARY 0
#define GHX_MODE_PARALLEL_COPY 1

/* executor kinds (ghx_exec_create) */
#define GHX_EXEC_DIRECT 0 /* local tags + remote tags pushed into peer fabs   */
#define GHX_EXEC_LOCAL 1  /* only tags whose src and dst rank are this rank   */
#define GHX_EXEC_PACK 2   /* remote tags of this rank -> per-peer send buffer */
#define GHX_EXEC_UNPACK 3 /* per-peer recv buffer -> remote tags into my fabs */
/* packed push: local tags + wide-row remote tags stored into peer fabs +
 * narrow-row remote tags (row bytes <= GHX_PACK_ROW_BYTES, default 128)
 * packed contiguously into the per-peer send slot (= the peer's mapped
 * receive buffer); the receiver then runs GHX_EXEC_UNPACK_PACKED. */
#define GHX_EXEC_PUSH_PACKED 4
#define GHX_EXEC_UNPACK_PACKED 5
/* the same pair with EVERY remote tag packed (no peer fab pointers needed):
 * used when fabs live in pinned host memory, which peers cannot IPC-map --
 * the sender's kernel reads its host fabs and stores the packed rows into
 * the peer's IPC-mapped DEVICE receive buffer; the receiver unpacks into
 * its own host fabs. */
#define GHX_EXEC_PUSH_PACKED_ALL 6
#define GHX_EXEC_UNPACK_PACKED_ALL 7
/* GHX_EXEC_PUSH_PACKED and GHX_EXEC_UNPACK_PACKED of one rank in ONE task
 * list and one launch (in-kernel synchronisation only, ghx_exec_run_synced):
 * the pushes first, then the local tags, then the unpacks of the receive
 * slabs; each peer's DONE is released as soon as this rank's pushes to it
 * are done, so the slabs that land early are unpacked while later pushes
 * are still in flight.  Send sizes: ghx_exec_buffer_elems; receive sizes:
 * ghx_exec_recv_elems. */
#define GHX_EXEC_EXCHANGE_PACKED 8
/* OR into the kind of a DIRECT / LOCAL FillBoundary executor whose tags are
 * all local: run the exchange in three phases (x faces; y faces extended over
 * the x ghosts; z faces extended over the x and y ghosts, reading the source
 * fab's ghosts filled by the earlier phases) with no edge / corner tags.
 * Same result bit for bit (fabs whose tags do not allow it keep theirs);
 * fewer, longer rows -- meant for fabs in host memory, where each PCIe
 * request costs.  Warps wait for each other between phases, so the grid
 * must be co-resident (host executors run 8 CTAs). */
#define GHX_EXEC_PHASED 0x100
/* Diagnostic (FillBoundary, local tags): OR GHX_EXEC_ONLY_XFACES to keep
 * only the x-face tags (ghost in x alone), GHX_EXEC_NO_XFACES to keep every
 * other tag -- the two halves of the exchange on the same storage layout,
 * timed separately by bench.py's direction split. */
#define GHX_EXEC_ONLY_XFACES 0x200
#define GHX_EXEC_NO_XFACES 0x400

typedef struct ghx_plan ghx_plan;
typedef struct ghx_exec ghx_exec;

const char *ghx_last_error(void);
int ghx_version(void);

/* ------------------------------------------------------------ box algebra */

/* Replaces the O(n^2) pairwise check in BoxArray.__init__ (mesh.py:203-205)
 * with a binned sweep.  *overlap_a = *overlap_b = -1 when disjoint, else the
 * lexicographically first overlapping pair (a < b). */
int ghx_boxes_disjoint(int64_t nboxes, const int64_t *boxes, int64_t *overlap_a,
                       int64_t *overlap_b);

/* ------------------------------------------------------------------ plans */

/* plan_build_fill_boundary (comm.py:289-309) minus the Python-side cache and
 * validation: dst targets = grow(box, ngrow), sources = valid boxes, the
 * (si == dj, shift == 0) pair excluded, pieces cut by box_diff against the
 * dst valid box (index_space.py:297-320); segments sorted by
 * (dst_fab, dst_lo, src_fab, shift) and grouped by (src_rank, dst_rank)
 * like CommPlan (comm.py:218-237).  periodic[d] != 0 marks periodic axes,
 * period[d] = geom.period (domain cell extent, index_space.py:371-374). */
int ghx_plan_build_fill_boundary(int64_t nboxes, const int64_t *boxes, const int64_t ngrow[3],
                                 const int32_t periodic[3], const int64_t period[3],
                                 const int32_t *rank_of, int32_t nranks, ghx_plan **out);

/* parallel_copy plan (comm.py:413-424): dst targets grow(dst_box, ngrow_dst),
 * sources grow(src_box, ngrow_src); periodic == NULL means geom=None (only
 * the zero shift, comm.py:253-254). */
int ghx_plan_build_parallel_copy(int64_t ndst, const int64_t *dst_boxes, const int64_t ngrow_dst[3],
                                 int64_t nsrc, const int64_t *src_boxes, const int64_t ngrow_src[3],
                                 const int32_t *periodic, const int64_t period[3],
                                 const int32_t *src_rank, const int32_t *dst_rank, int32_t nranks,
                                 ghx_plan **out);

void ghx_plan_free(ghx_plan *plan);
int64_t ghx_plan_num_segments(const ghx_plan *plan);
/* rows of 13 int64: src_fab dst_fab dlo0 dlo1 dlo2 dhi0 dhi1 dhi2 s0 s1 s2
 * src_rank dst_rank, in CommPlan sort order (src box = dst box - shift). */
int ghx_plan_get_segments(const ghx_plan *plan, int64_t *rows);
/* number of write tags after last-writer-wins clipping (== segments unless
 * destinations overlap: nodal data or ngrow_src > 0). */
int64_t ghx_plan_num_write_tags(const ghx_plan *plan);
/* per (src_rank, dst_rank) cell totals of the reference segments:
 * out[(s * nranks + d)] = cells (local pairs s == d included). */
int ghx_plan_pair_cells(const ghx_plan *plan, int64_t *out);

/* ------------------------------------------------------------- executors */

/* Compile the plan for one rank and one storage layout into a device tag
 * table (one fused launch per run).  src_fab_boxes / dst_fab_boxes: storage
 * (grown) box of every src / dst fab (nsrc*6, ndst*6), ncomp_total the
 * fab's component count; components [scomp, scomp+ncomp) of src land in
 * [dcomp, dcomp+ncomp) of dst.  elem_bytes: 4 or 8. */
int ghx_exec_create(const ghx_plan *plan, int32_t rank, int32_t kind, const int64_t *src_fab_boxes,
                    int32_t src_ncomp_total, const int64_t *dst_fab_boxes, int32_t dst_ncomp_total,
                    int32_t scomp, int32_t dcomp, int32_t ncomp, int32_t elem_bytes, int32_t device,
                    ghx_exec **out);
void ghx_exec_free(ghx_exec *ex);

/* Run the fused copy kernel.  ptrs: device-accessible base pointers, laid
 * out as [nsrc src fabs][ndst dst fabs][nranks send buffers][nranks recv
 * buffers]; entries never referenced by this rank's tags may be NULL.
 * Base pointers must be 16-byte aligned. */
int ghx_exec_run(ghx_exec *ex, void *const *ptrs, int64_t nptrs, void *stream);

/* Pinned bindings.  ghx_exec_bind resolves a pointer table into the
 * executor's own descriptor copy once (stream-ordered; completed before it
 * returns unless the stream is capturing) and returns a binding id that
 * ghx_exec_run_bound launches with no host table work.  A pinned binding is
 * never recycled by ghx_exec_run, so CUDA graphs that captured its launch
 * stay valid; ghx_exec_unbind releases the pin.  Every binding has its own
 * scheduler counter, so different bindings of one executor may run on
 * different streams concurrently; ONE binding must not be enqueued on two
 * streams at once. */
int ghx_exec_bind(ghx_exec *ex, void *const *ptrs, int64_t nptrs, void *stream, int64_t *binding);
int ghx_exec_run_bound(ghx_exec *ex, int64_t binding, void *stream);
int ghx_exec_unbind(ghx_exec *ex, int64_t binding);

/* Introspection: tags, warp tasks, elements moved per run, algorithmic
 * bytes (read + write) per run, per-peer buffer elements (out[nranks]). */
int ghx_exec_info(const ghx_exec *ex, int64_t *ntags, int64_t *ntasks, int64_t *elems,
                  int64_t *alg_bytes);
int ghx_exec_buffer_elems(const ghx_exec *ex, int64_t *per_peer);
/* out[8] = tags, warp tasks, elements, algorithmic bytes, tags in mirror
 * pairs, tags in sector-swap pairs, grid blocks, load flavour. */
int ghx_exec_detail(const ghx_exec *ex, int64_t out[8]);

/* Seam-chunk ("ring") tasks for x-face sector swaps of periodic x-lines:
 * each 64-byte row seam is read and written with one coalesced access
 * (fewer, larger transactions: meant for fabs in host memory over PCIe;
 * on HBM the sector-swap chains are faster).  Only before the first run. */
int ghx_exec_set_ring(ghx_exec *ex, int32_t on);

/* TMA bulk-row tasks (cp.async.bulk through shared memory) for wide rows
 * (256 B - 8 KB, 16-byte aligned).  Default: on for FillBoundary of large
 * fabs; for ParallelCopy only when the caller guarantees that no source
 * byte is written by the same run (distinct MultiFabs).  Only before the
 * first run. */
int ghx_exec_set_bulk(ghx_exec *ex, int32_t on);

/* Task mix: out[6] = copy tasks, sector-swap tasks, x-line chain tasks,
 * seam-chunk ring tasks, ring mode on, fab-local order on. */
int ghx_exec_task_kinds(const ghx_exec *ex, int64_t out[6]);

/* Phased executors: out[4] = phased (0/1), first task of phase 1, first task
 * of phase 2, device tags. */
int ghx_exec_phases(const ghx_exec *ex, int64_t out[4]);

/* Unpack executors of a FillBoundary: how many x-face ghost tags run as
 * sector fills (each 16-byte ghost half stored with the valid half of its
 * 32-byte sector, read from the same fab, so no partial-sector writes;
 * GHX_SECTOR_FILL=0 at create time turns it off). */
int ghx_exec_sector_fills(const ghx_exec *ex, int64_t *ntags);

/* Per-peer receive-buffer elements of a GHX_EXEC_EXCHANGE_PACKED executor
 * (what each peer packs for this rank); other kinds: the unpack kinds'
 * buffer sizes, zeros for the rest.  per_peer: nranks entries. */
int ghx_exec_recv_elems(const ghx_exec *ex, int64_t *per_peer);

/* Launch-time tuning knob (warps per block * blocks): 0 = default. */
int ghx_exec_set_grid(ghx_exec *ex, int32_t blocks, int32_t threads);

/* -------------------------------------------------------------- devices */

int ghx_device_alloc(int32_t device, size_t bytes, void **out);
int ghx_device_free(void *ptr);
int ghx_host_alloc(size_t bytes, void **out); /* pinned + mapped */
int ghx_host_free(void *ptr);
int ghx_memset_u64(void *ptr, uint64_t value, size_t count, void *stream);
int ghx_enable_peer_access(int32_t device, int32_t peer);
int ghx_ipc_get_handle(void *ptr, uint8_t handle[64]);
int ghx_ipc_open_handle(int32_t device, const uint8_t handle[64], void **out);
/* Byte offset of ptr inside its device allocation (IPC maps whole allocations). */
int ghx_alloc_offset(const void *ptr, uint64_t *offset);
int ghx_ipc_close_handle(void *ptr);
int ghx_stream_sync(void *stream);

/* Cross-rank device barrier: rank writes `epoch` into flags[p][rank] of
 * every peer p (system-scope release), then spins until its own
 * flags[rank][p] >= epoch for all p (acquire).  flag_ptrs[p] is rank p's
 * flag array (nranks uint64) as mapped in this process. */
int ghx_signal_barrier(uint64_t *const *flag_ptrs, int32_t rank, int32_t nranks, uint64_t epoch,
                       void *stream);
/* In-kernel synchronisation of process-mode exchanges (one GPU per rank),
 * replacing the barrier -> push -> barrier -> unpack sequence: rank p's
 * flag array holds 3*nranks uint64 slots ([0,n) ghx_signal_barrier, [n,2n)
 * READY, [2n,3n) DONE).  ghx_exec_set_sync gives the executor every rank's
 * array as mapped here.  ghx_exec_run_synced launches a push executor
 * (DIRECT / PUSH_PACKED*) so that it signals READY to every peer on entry,
 * runs its remote tasks (ordered first) only after the destination peer's
 * READY, and signals DONE once all its pushes are visible; or a packed
 * unpack executor so that each peer's receive slab is unpacked as soon as
 * that peer's DONE lands and the kernel completes only after every peer's
 * DONE.  ghx_exec_sync_wait is the DONE wait alone (direct mode exit).
 * Epochs must increase and be identical on every rank. */
int ghx_exec_set_sync(ghx_exec *ex, uint64_t *const *flag_arrays, int32_t rank, int32_t nranks);
int ghx_exec_run_synced(ghx_exec *ex, int64_t binding, uint64_t epoch, void *stream);
int ghx_exec_sync_wait(ghx_exec *ex, uint64_t epoch, void *stream);

/* Number of device barriers (this process, current device) that gave up
 * after GHX_BARRIER_TIMEOUT_S seconds (default 30) instead of hanging;
 * synchronous read, -1 on error. */
int64_t ghx_barrier_timeouts(void);

/* Synthetic input generator (bench / tests): valid cells of the fab get
 * splitmix64(seed ^ lin(i,j,k,c)) mapped to [0,1) (see oracle/inputs.py),
 * every other storage cell gets the signalling-NaN poison. */
int ghx_fill_hash(void *fab, const int64_t fab_box[6], int32_t ncomp, const int64_t valid_box[6],
                  const int64_t domain_box[6], uint64_t seed, int32_t elem_bytes, void *stream);

/* Expected state after a FillBoundary of a field filled by ghx_fill_hash:
 * every storage cell whose periodically wrapped coordinate lies in the
 * domain holds the hash of the wrapped cell, every other cell the poison.
 * (Size-independent parity property for full-size configurations.) */
int ghx_fill_hash_wrapped(void *fab, const int64_t fab_box[6], int32_t ncomp, const int64_t domain_box[6],
                          const int32_t periodic[3], uint64_t seed, int32_t elem_bytes, void *stream);

/* ------------------------------------------------------------ index copy */

/* index_mapped_copy's data movement (reference comm.py:465-560): for every
 * cell, ncomp raw words from src to dst.  d_rows: device array of ncells
 * rows {src byte address, dst byte address, src component stride (bytes),
 * dst component stride (bytes)}; addresses may be peer or IPC mappings. */
int ghx_index_copy(const int64_t *d_rows, int64_t ncells, int32_t ncomp, int32_t elem_bytes, void *stream);

/* ----------------------------------------------------------------- arena */

/* Pooled arena (reference arena.py:87-197): slabs + LIFO free lists per
 * (padded size, alignment); kind SYSTEM makes one allocation per request.
 * memory: device HBM (device = CUDA ordinal), pinned+mapped host, or plain
 * host memory (host-only tests).  Thread-safe.  A zero-byte allocation
 * returns NULL; freeing a pointer that is not a live block (double free)
 * returns GHX_EOVERLAP.  Stats: reserved, in-use (padded), alloc calls,
 * slab growths. */
#define GHX_ARENA_POOLED 0
#define GHX_ARENA_SYSTEM 1
#define GHX_ARENA_DEVICE 0
#define GHX_ARENA_PINNED 1
#define GHX_ARENA_HOST 2
typedef struct ghx_arena ghx_arena;
int ghx_arena_create(int32_t kind, int32_t memory, int32_t device, size_t capacity_bytes, ghx_arena **out);
int ghx_arena_alloc(ghx_arena *a, size_t nbytes, size_t align, void **out);
int ghx_arena_free(ghx_arena *a, void *ptr);
/* Stream-ordered free: the block is recycled once the work queued so far on
 * every given stream (cudaStream_t) has completed; nstreams == 0 frees now.
 * Parked blocks still count as in use; ghx_arena_poll recycles the finished
 * ones and reports how many are still parked. */
int ghx_arena_free_after(ghx_arena *a, void *ptr, void *const *streams, int32_t nstreams);
int ghx_arena_poll(ghx_arena *a, int64_t *parked);
int ghx_arena_block_size(const ghx_arena *a, const void *ptr, size_t *padded);
int ghx_arena_stats(const ghx_arena *a, int64_t out[4]);
void ghx_arena_destroy(ghx_arena *a);

/* Number of fused-copy kernel launches issued by this process. */
int64_t ghx_launch_count(void);

/* ------------------------------------------------ coarse/fine transfers */

#define GHX_INTERP_PC 0     /* amr.PIECEWISE_CONSTANT */
#define GHX_INTERP_LINEAR 1 /* amr.LINEAR: unlimited centred slopes */

/* One interp_box job (reference amr.py:269-314): fill `region` (fine
 * index space) of the fine fab from the coarse fab.  Boxes are the fabs'
 * storage boxes, padded to 3 axes (lo = hi = 0).  Requires region inside
 * fine_box and coarsen(region) (grown by 1 on axes < spacedim for LINEAR)
 * inside crse_box, else GHX_EINVAL ("insufficient coarse data"). */
typedef struct {
  const void *crse;
  int64_t crse_box[6];
  void *fine;
  int64_t fine_box[6];
  int64_t region[6];
} ghx_interp_job;

/* Every job in ONE launch on `stream`; ncomp components (both fabs), ratio
 * per axis (1 on axes >= spacedim), float64 or float32 storage.  Results
 * are bit-identical to numpy's evaluation order in interp_box. */
int ghx_interp(const ghx_interp_job *jobs, int64_t njobs, int32_t ncomp, const int32_t ratio[3], int32_t spacedim,
               int32_t scheme, int32_t elem_bytes, void *stream);

/* One restriction job of average_down (amr.py:251-264): every coarse cell
 * of `region` (coarse index space) becomes the mean of its ratio^D fine
 * children (summed in (oz, oy, ox) order, divided by ratio^spacedim). */
typedef struct {
  const void *fine;
  int64_t fine_box[6];
  void *crse;
  int64_t crse_box[6];
  int64_t region[6];
} ghx_avgdown_job;

int ghx_average_down(const ghx_avgdown_job *jobs, int64_t njobs, int32_t ncomp, const int32_t ratio[3],
                     int32_t spacedim, int32_t elem_bytes, void *stream);

/* Prepared transfers: the job table is validated and uploaded once
 * (device `device`), each ghx_xfer_run is one launch on `stream` with no
 * host-side work (fill_patch / average_down cache one per plan).  Fab
 * pointers are baked in: the fabs must outlive the handle. */
typedef struct ghx_xfer ghx_xfer;
int ghx_interp_prepare(const ghx_interp_job *jobs, int64_t njobs, int32_t ncomp, const int32_t ratio[3],
                       int32_t spacedim, int32_t scheme, int32_t elem_bytes, int32_t device, ghx_xfer **out);
int ghx_average_down_prepare(const ghx_avgdown_job *jobs, int64_t njobs, int32_t ncomp, const int32_t ratio[3],
                             int32_t spacedim, int32_t elem_bytes, int32_t device, ghx_xfer **out);
/* One heat-equation step (reference heat.py:172-189) over `region` of each
 * job: dst = src + sum_d coef[d] * ((src[+e_d] - 2 src) + src[-e_d]) for
 * d < spacedim, component 0, numpy's operation order (bit-exact).  src must
 * hold the region grown by one cell (its ghosts filled). */
typedef struct {
  const void *src;
  int64_t src_box[6];
  void *dst;
  int64_t dst_box[6];
  int64_t region[6];
} ghx_stencil_job;
#define GHX_ADVANCE_TILES 0 /* 32x8 (x,y) tiles marching z: thick regions */
#define GHX_ADVANCE_CELLS 1 /* one thread per cell: thin shells */
int ghx_advance_prepare(const ghx_stencil_job *jobs, int64_t njobs, const double coef[3], int32_t spacedim,
                        int32_t elem_bytes, int32_t layout, int32_t device, ghx_xfer **out);

int ghx_xfer_run(ghx_xfer *x, void *stream);
int64_t ghx_xfer_cells(const ghx_xfer *x); /* cells written per run */
void ghx_xfer_free(ghx_xfer *x);

/* Number of interp / average_down launches issued by this process. */
int64_t ghx_amr_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* GHOSTX_H */
