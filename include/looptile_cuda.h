/*
 * looptile_cuda.h — C ABI of libltcuda.so, the B200 (sm_100a) sparse-tiling
 * inspector/executor for unstructured-mesh loop chains.
 *
 * The reference (`looptile`, pure Python, /root/reference/pkg/src/looptile) has
 * no native boundary; its plugin surface is the Python API re-exported in
 * `looptile/__init__.py:9-21`.  Every entry point below replaces one reference
 * function (cited per declaration) and is bound from Python by
 * paper_1708_03183_b200/_lib.py (ctypes).  Plain pointers and sizes only:
 * arrays marked "device" live in HBM (caller-owned unless stated), arrays
 * marked "host" in host memory.  Element ids are int32 on the device (the
 * reference uses int64; ids < 2^31 are enforced at chain build time).
 *
 * Errors: every function returns LT_OK (0) or a negative LT_E_* code, one per
 * exception class of `looptile/errors.py:4-33`; lt_last_error() returns the
 * thread-local message.  There is no CPU fallback: without a usable CUDA
 * device every compute entry point fails with LT_E_CUDA.
 *
 * Threading/ordering: one lt_ctx per device; calls are ordered on the
 * context's stream (lt_ctx_set_stream) and asynchronous unless documented as
 * synchronous.  A handle must not be used from two host threads at once.
 */
#ifndef LOOPTILE_CUDA_H
#define LOOPTILE_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LT_ABI_VERSION 2

/* status codes (errors.py:4-33) */
#define LT_OK                 0
#define LT_E_INVALID_CHAIN   -1  /* InvalidChainError */
#define LT_E_DEPTH_EXCEEDED  -2  /* DepthExceededError */
#define LT_E_INSPECTION      -3  /* InspectionError */
#define LT_E_COLORING_LIMIT  -4  /* ColoringLimitError */
#define LT_E_EXECUTION       -5  /* ExecutionError */
#define LT_E_STALE_SCHEDULE  -6  /* StaleScheduleError */
#define LT_E_PARTITION       -7  /* PartitionBugError */
#define LT_E_VALUE           -8  /* ValueError (e.g. tile size < 1, inspector.py:191) */
#define LT_E_CUDA            -9  /* CUDA runtime failure / no device */

/* access modes (chain.py:21-24, plus RW) */
#define LT_READ  0
#define LT_WRITE 1
#define LT_INC   2
#define LT_RW    3

/* execution modes (inspector.py:25-28) */
#define LT_SEQUENTIAL  0
#define LT_SHARED      1
#define LT_DISTRIBUTED 2

/* regions (chain.py:38-43) */
#define LT_CORE     0
#define LT_BOUNDARY 1
#define LT_NONEXEC  2

/* executor phases (executor.py:205-245) */
#define LT_PHASE_CORE     1
#define LT_PHASE_BOUNDARY 2

typedef struct lt_ctx lt_ctx;
typedef struct lt_schedule lt_schedule;

/* IterationSpace (chain.py:46-74): ids 0..total-1 stored core|boundary|nonexec */
typedef struct {
    int64_t core;
    int64_t boundary;
    int64_t nonexec;
} lt_space;

/* MeshMap (chain.py:77-102): values = device int32[n_source*arity] */
typedef struct {
    int32_t source;      /* index into lt_chain.spaces */
    int32_t target;
    int32_t arity;
    int32_t reserved;
    const int32_t *values;
} lt_map;

/* Descriptor (chain.py:141-150): map = index into lt_chain.maps, -1 = direct */
typedef struct {
    int32_t map;
    int32_t mode;        /* LT_READ .. LT_RW */
} lt_desc;

/* Loop (chain.py:153-158): kernel = native kernel id from lt_kernel_lookup */
typedef struct {
    int32_t space;
    int32_t n_desc;
    int32_t kernel;
    int32_t reserved;
    const lt_desc *desc;
} lt_loop;

/* LoopChain (chain.py:161-187); validation stays host-side (build_chain) */
typedef struct {
    int32_t n_spaces;
    int32_t n_maps;
    int32_t n_loops;
    int32_t depth;
    const lt_space *spaces;
    const lt_map *maps;
    const lt_loop *loops;
} lt_chain;

/* Dataset bound to one descriptor (executor.py:25-39, KernelBinding :64-69) */
typedef struct {
    double *values;      /* device float64[n_elements*vpe], element-major */
    int64_t n_elements;  /* space total of the dataset */
    int32_t vpe;         /* values_per_element */
    int32_t reserved;
} lt_arg;

/* Schedule summary (inspector.py:104-179, InspectionStats :83-101) */
typedef struct {
    int32_t mode;
    int32_t n_loops;
    int32_t n_tiles;     /* including the trailing non-exec tile */
    int32_t n_core_tiles;
    int32_t n_boundary_tiles;
    int32_t rounds;      /* recolor_rounds */
    int32_t n_colors;
    int32_t reserved;
    double partition_s;
    double coloring_s;
    double projection_tiling_s;
    double local_maps_s;
    double total_s;
} lt_schedule_info;

/* ExecutionReport counters (executor.py:72-95) */
typedef struct {
    int32_t launches;    /* kernel launches issued by this call */
    int32_t n_colors;    /* colour phases executed */
    int64_t elements;    /* element visits (sum over loops) */
    int32_t staged;      /* 0: global-memory tiles, 1: staged per colour, 2: staged dataflow */
    int32_t smem_bytes;  /* dynamic shared memory per CTA */
    int32_t wave_order;  /* dataflow queue: 1 wavefront (L2-local) order, 0 colour-major */
    int32_t wide_build;  /* dataflow: 1 when the 128-register build ran (<= 4 CTAs/SM) */
} lt_exec_info;

/* ---- library / context ---------------------------------------------------- */
int         lt_abi_version(void);
const char *lt_last_error(void);
int lt_ctx_create(int device, lt_ctx **out);
int lt_ctx_destroy(lt_ctx *ctx);
/* stream = cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream) */
int lt_ctx_set_stream(lt_ctx *ctx, void *stream);
int lt_ctx_synchronize(lt_ctx *ctx);
/* drop cached device state derived from a map buffer before it is freed */
int lt_ctx_forget_map(lt_ctx *ctx, const int32_t *values);

/* ---- native kernel registry (replaces KernelRegistry bodies, executor.py:46-61,
 *      and the preset bodies of problems.py:49-64) --------------------------- */
/* name -> id and argument count; LT_E_EXECUTION if unknown */
int lt_kernel_lookup(const char *name, int32_t *kernel_id, int32_t *nargs);
int lt_kernel_count(void);
const char *lt_kernel_name(int32_t kernel_id);
/* per-context parameter block of a kernel (e.g. DG operator tables, dt);
 * host float64[n] copied to the device */
int lt_ctx_set_kernel_params(lt_ctx *ctx, int32_t kernel_id, const double *host, int64_t n);

/* ---- inspector (inspector.py:433-495 and its steps) ------------------------ */
/* invert_map (chain.py:118-135): offsets device int32[n_target+1],
 * sources device int32[n_source*arity], each segment ascending */
int lt_invert_map(lt_ctx *ctx, const int32_t *values, int64_t n_source, int32_t arity,
                  int64_t n_target, int32_t *offsets, int32_t *sources);
/* inspect_chain (inspector.py:433): full GPU inspection, synchronous */
int lt_inspect(lt_ctx *ctx, const lt_chain *chain, int64_t tile_size, int32_t mode,
               lt_schedule **out);
/* Schedule built from host iteration lists (e.g. the CPU oracle's or the
 * reference's schedule): colors/regions host int32[n_tiles]; for loop j,
 * offsets[j] host int32[n_tiles+1] and elements[j] host int32[space total] */
int lt_schedule_import(lt_ctx *ctx, const lt_chain *chain, int32_t mode, int32_t n_tiles,
                       const int32_t *colors, const int32_t *regions, int32_t rounds,
                       const int32_t *const *offsets, const int32_t *const *elements,
                       lt_schedule **out);
int lt_schedule_info_get(const lt_schedule *s, lt_schedule_info *info);
/* host outputs: colors/regions int32[n_tiles] */
int lt_schedule_tiles(const lt_schedule *s, int32_t *colors, int32_t *regions);
/* host outputs: offsets int32[n_tiles+1], elements int32[space total]
 * (Tile.iteration_lists, inspector.py:38-50 / assign :385-391) */
int lt_schedule_lists(const lt_schedule *s, int32_t loop, int32_t *offsets, int32_t *elements);
/* device view of the per-element tile assignment (Schedule.tile_of) */
int lt_schedule_tile_of(const lt_schedule *s, int32_t loop, const int32_t **device_sigma,
                        int64_t *n);
/* host output int32[space total * arity]: compute_local_maps (inspector.py:397-418)
 * for the loop's map (index into lt_chain.maps); LT_E_VALUE if the loop has no such map */
int lt_schedule_local_map(const lt_schedule *s, int32_t loop, int32_t map, int32_t *out);
int lt_schedule_destroy(lt_schedule *s);

/* ---- step-level inspector (the public steps of inspector.py) -----------------
 * Tile pairs are encoded (a << 32) | b with a < b; *n_pairs receives the
 * total, at most `capacity` are written to `pairs` (host). */
/* partition_seed (inspector.py:185-205): sigma device int32[space total] */
int lt_partition_seed(lt_ctx *ctx, const lt_space *space, int64_t tile_size, int32_t *sigma,
                      int32_t *n_core_tiles, int32_t *n_boundary_tiles);
/* assign (inspector.py:385-391): device offsets int32[n_tiles+1], elements int32[n] */
int lt_assign(lt_ctx *ctx, const int32_t *sigma, int64_t n, int32_t n_tiles, int32_t *offsets,
              int32_t *elements);
/* _seed_adjacency (inspector.py:208-225): tiles sharing a target of the seed map */
int lt_seed_adjacency(lt_ctx *ctx, const int32_t *map_values, int64_t n_source, int32_t arity,
                      int64_t n_target, const int32_t *sigma, int32_t n_tiles, int64_t *pairs,
                      int64_t capacity, int64_t *n_pairs);
/* color_tiles (inspector.py:228-263), host only: regions host int32[n_tiles],
 * pairs = adjacency (seed adjacency + fake connections), colors host out */
int lt_color_tiles(int32_t n_tiles, const int32_t *regions, int32_t mode, const int64_t *pairs,
                   int64_t n_pairs, int32_t *colors);
/* project (inspector.py:266-316) of loop `loop`: phi[s] = device int32[space s total]
 * per chain space, present[s] (host) says whether phi[s] holds a projection;
 * both are updated; conflict pairs returned */
int lt_project(lt_ctx *ctx, const lt_chain *chain, int32_t loop, const int32_t *sigma,
               const int32_t *colors, int32_t n_tiles, int32_t *const *phi, int32_t *present,
               int64_t *pairs, int64_t capacity, int64_t *n_pairs);
/* tile_loop (inspector.py:319-382): sigma_out device int32[space total];
 * tne >= 0 forces non-exec elements to tile tne (inspect_chain :480);
 * detect != 0 runs the second (conflict) sweep */
int lt_tile_loop(lt_ctx *ctx, const lt_chain *chain, int32_t loop, int32_t *const *phi,
                 const int32_t *present, const int32_t *colors, int32_t n_tiles, int32_t tne,
                 int32_t *sigma_out, int32_t detect, int64_t *pairs, int64_t capacity,
                 int64_t *n_pairs);

/* compute_local_maps (inspector.py:397-418): out[p*arity+k] = map[elements[p]*arity+k] */
int lt_gather_rows(lt_ctx *ctx, const int32_t *map_values, int32_t arity, const int32_t *elements,
                   int64_t n, int32_t *out);

/* ---- executor (executor.py:163-245) ---------------------------------------- */
/* args: flat lt_arg array, loop-major, one per descriptor.
 * execute_schedule: run the selected phases (LT_PHASE_CORE|LT_PHASE_BOUNDARY);
 * the caller brackets them with its halo exchange begin()/end() */
int lt_execute(lt_ctx *ctx, lt_schedule *s, const lt_chain *chain, const lt_arg *args,
               int32_t phases, int32_t use_local_maps, lt_exec_info *info);
/* execute_schedule repeated `repeats` times back to back (a time-stepping loop
 * over the same chain, no halo exchange in between); the dataflow executor
 * overlaps consecutive repeats tile by tile */
int lt_execute_repeat(lt_ctx *ctx, lt_schedule *s, const lt_chain *chain, const lt_arg *args,
                      int32_t repeats, int32_t use_local_maps, lt_exec_info *info);
/* Build the execution plan (tile programs, dependency graph, queue) that a
 * later lt_execute / lt_execute_repeat with the same arguments uses, without
 * launching anything or touching the datasets.  No reference counterpart: the
 * reference executor has no plan (executor.py:185-245); this splits its
 * one-time validation from the steady-state call so time-stepping drivers and
 * CUDA-graph capture never run the chain just to build the plan. */
int lt_prepare(lt_ctx *ctx, lt_schedule *s, const lt_chain *chain, const lt_arg *args,
               int32_t phases, int32_t repeats, int32_t use_local_maps, lt_exec_info *info);
/* execute_untiled: loops in order, elements ascending (executor.py:163-169) */
int lt_execute_untiled(lt_ctx *ctx, const lt_chain *chain, const lt_arg *args,
                       lt_exec_info *info);

/* Legality of a schedule (reference pkg/tests/legality.py:15-151, the
 * brute-force dependence oracle the reference's property tests use): counts
 * the distinct cross-loop dependence pairs (flow/anti/output through a shared
 * (space, element), not both direct) whose later element runs in a different
 * tile of a colour not above the earlier one's, and the reduction pairs
 * (same loop, mapped increments of one key) split over distinct tiles of equal
 * colour.  Runs on the GPU at any size; overflow = 1 when more than 2^20
 * violations were found (counts are then lower bounds). */
int lt_check_legality(lt_ctx *ctx, const lt_schedule *s, const lt_chain *chain,
                      int64_t *n_pairs, int64_t *n_reductions, int32_t *overflow);

/* ---- halo exchange packing (distsim.py:48-81) ------------------------------ */
/* out[i*vpe + c] = values[rows[i]*vpe + c] for i < n_rows (device arrays) */
int lt_halo_pack(lt_ctx *ctx, const double *values, int32_t vpe, const int32_t *rows,
                 int64_t n_rows, double *out);
/* values[rows[i]*vpe + c] = in[i*vpe + c] */
int lt_halo_unpack(lt_ctx *ctx, double *values, int32_t vpe, const int32_t *rows,
                   int64_t n_rows, const double *in);

/* ---- host-side data-layout pass (mesh.py:123-145), no device needed ------- */
/* Reverse Cuthill-McKee over a CSR graph (neighbour lists sorted ascending);
 * order_out[k] = old id placed k-th; LT_E_VALUE if disconnected */
int lt_rcm_order(int64_t n, const int64_t *offsets, const int64_t *neighbours,
                 int64_t *order_out);

#ifdef __cplusplus
}
#endif

#endif /* LOOPTILE_CUDA_H */
