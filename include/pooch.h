/* pooch.h -- C ABI of the B200-native PoocH out-of-core training-step executor.
 *
 * PoocH (arXiv 1907.05013, "Profiling-based out-of-core Hybrid method") trains a CNN whose
 * feature maps exceed device memory by classifying every feature map as keep / swap /
 * recompute (Sec. 4.1.1) from a plan built by simulating a profiled iteration
 * (Sec. 4.1.2). The flow is "1. Profiling  2. Classification  3. Execution"
 * (P:L169-173); the calls below follow it:
 *
 *   pooch_create -> pooch_set_budget -> pooch_set_streams -> [pooch_set_comm]
 *     -> pooch_profile (Sec. 4.2) -> pooch_plan (Sec. 4.4) -> pooch_train_step* (execution)
 *
 * Citations: P:Lnnn = PAPER.md line (section / equation named alongside).
 *
 * Conventions for every function:
 *  - Returns pooch_status; nothing throws or aborts across the ABI. On failure the
 *    per-context message is available from pooch_last_error (ctx-less calls: pass NULL).
 *  - Pointers are plain host or device pointers as stated per argument; sizes are bytes
 *    unless stated otherwise. Activations are NHWC fp32, conv weights KRSC fp32
 *    ([Cout][R][S][Cin], Cin padded to a multiple of 4), FC weight [Cout][Cin].
 *  - Ownership: the caller owns the device arena, the pinned host arena and the CUDA
 *    streams and keeps them alive until pooch_destroy; the library never calls
 *    cudaMalloc / cudaHostAlloc. The library owns the context, profile, plan, schedule,
 *    CUDA events and the NCCL communicator.
 *  - A context is single-threaded: one context per device / rank.
 *  - Asynchronous CUDA faults surface as POOCH_ECUDA at the next call that synchronises.
 */
#ifndef POOCH_H
#define POOCH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pooch_ctx pooch_ctx;

typedef enum {
  POOCH_OK = 0,
  POOCH_EUSAGE = 1,      /* bad argument / call order */
  POOCH_EINFEASIBLE = 2, /* no plan fits the budget (memory must never exceed capacity) */
  POOCH_ENOPLAN = 3,     /* train_step without a current plan (budget / comm changed since) */
  POOCH_ECUDA = 4,       /* CUDA runtime error; message has the runtime's string */
  POOCH_ENCCL = 5        /* NCCL error */
} pooch_status;

/* The three classes of a feature map (Sec. 4.1.1). */
typedef enum { POOCH_KEEP = 0, POOCH_SWAP = 1, POOCH_RECOMPUTE = 2 } pooch_class;

/* Planning strategies: PoocH itself (Sec. 4.4) and the comparison points of Sec. 5.1-5.2
 * (P:L352-356). EXHAUSTIVE enumerates all 2*3^(n-1) classifications (n <= 12). */
typedef enum {
  POOCH_STRAT_POOCH = 0,
  POOCH_STRAT_INCORE = 1,
  POOCH_STRAT_SWAP_ALL_NAIVE = 2,
  POOCH_STRAT_SWAP_ALL = 3,
  POOCH_STRAT_SWAP_OPT = 4,
  POOCH_STRAT_SUPERNEURONS = 5, /* static rule of P:L395-400, scheduled with POOCH_SCHED_SN */
  POOCH_STRAT_EXHAUSTIVE = 6,
  POOCH_STRAT_FIXED = 7
} pooch_strategy;

/* Swap-in scheduling (Sec. 4.3): EAGER = "when there is room in the GPU memory";
 * NAIVE = starts with the computation just before its first user.
 * EAGER, as built (DESIGN.md Reading 9): swap-ins are issued in need order once the forward pass
 * has ended, and "room" is live + bytes + H(m) <= budget, where H(m) is the peak extra memory the
 * compute program needs before the map's first use -- stricter than issuing whenever the H2D lane
 * is free and live + bytes fits (which can let a prefetch take memory an earlier backward task
 * needs and deadlock); the simulator, the oracle and the executor all use this rule. */
typedef enum { POOCH_SCHED_EAGER = 0, POOCH_SCHED_NAIVE = 1, POOCH_SCHED_SN = 2 } pooch_sched;
/* POOCH_SCHED_SN: SuperNeurons' rule, "each swap-in starts simultaneously with the computation
 * of the immediately preceding convolution layer". */

/* ------------------------------------------------------------------ network description */
/* One fused executor task. A task's output is one feature map. */
typedef enum {
  POOCH_L_CONV = 0,      /* y = conv(x, W), no bias                     bwd reads {x}      */
  POOCH_L_BNRELU = 1,    /* y = relu(BN(c)), training-mode BN           bwd reads {c}      */
  POOCH_L_TAIL_PROJ = 2, /* y = relu(BN3(c3) + BNp(p))  (bottleneck end) bwd reads {c3, p}  */
  POOCH_L_TAIL_ID = 3,   /* y = relu(BN3(c3) + x)                        bwd reads {c3, x}  */
  POOCH_L_MAXPOOL = 4,   /* y = maxpool(x)                               bwd reads {x}      */
  POOCH_L_AVGPOOL = 5,   /* y = mean_hw(x)                               bwd reads {}       */
  POOCH_L_FC_CE = 6,     /* z = flat_hwc(x) W^T + b, softmax-CE loss     bwd reads {x, z}   */
  POOCH_L_UPCONV = 7,    /* y = transposed conv k2 s2 of x (3D U-Net up-sampling)  bwd reads {x} */
  POOCH_L_HEAD_CE = 8,   /* z = x W^T + b per voxel, softmax-CE averaged over voxels  bwd reads {x, z} */
  POOCH_L_BNRELU_CONV = 9, /* y = conv(relu(BN(c)), W): BN-ReLU applied to the conv's operand on
                             load, relu(BN(c)) never stored   bwd reads {c} */
  /* AlexNet: */
  POOCH_L_CONV_RELU = 10,   /* y = relu(conv(x, W) + b), bias per output channel   bwd reads {x, y} */
  POOCH_L_LRN = 11,         /* y = x / (2 + 1e-4 / 5 * sum_{|c'-c| <= 2} x_c'^2)^0.75 (local response
                               normalisation across channels)                      bwd reads {x}    */
  POOCH_L_FC_RELU_DROP = 12 /* y = dropout(relu(flat_hwc(x) W^T + b)), inverted dropout with a
                               counter-based mask (pooch_set_rng); k = drop probability in percent,
                               output [batch][cout] (hout = wout = 1)           bwd reads {x, y}    */
} pooch_layer_kind;
/* POOCH_L_BNRELU_CONV: c (in0) is a conv output with this task as its only consumer; 2D, single
 * input, cin a multiple of 32, stride <= 2. name = "<bn name>+<conv name>": the BN's gamma /
 * beta are named after the first part, the conv weight after the second. */
/* A POOCH_L_CONV with in1 >= 0 reads the channel concatenation [in0, in1] in place (the
 * U-Net's skip connection): cin = cout(in0) + cout(in1), both multiples of 32.
 * 3D networks (io.in_d > 0, batch 1): every conv is k x k x k; maxpool is k2 s2 p0 over 2^3
 * windows; UPCONV has k = stride = 2 and doubles each spatial extent. */

typedef struct {
  int32_t kind;          /* pooch_layer_kind */
  int32_t in0, in1;      /* producer task ids (< this id); -1 = network input / unused */
  int32_t cin;           /* input channels as stored (padded to a multiple of 4) */
  int32_t cout, hout, wout; /* output map shape per image (C, H, W) */
  int32_t k, stride, pad;   /* conv / pool geometry */
  char name[48];
  int32_t dout;             /* output depth of a 3D network's map (0 in 2D networks) */
  int32_t groups;           /* POOCH_L_CONV: 0 / 1 dense, > 1 grouped (see pooch_conv_desc.groups) */
  int32_t stride_d;         /* 3D POOCH_L_CONV: depth stride (0 = stride) */
} pooch_layer_desc;

typedef struct {
  int32_t batch;         /* per-rank batch */
  int32_t in_c, in_h, in_w; /* network input, in_c padded to a multiple of 4 */
  int32_t classes;
  int32_t in_d;          /* 0: 2D network (NHWC input); > 0: 3D network, input [batch, in_d, in_h, in_w, in_c] */
} pooch_io_desc;

/* Built-in workloads of BASELINE.json: 0 = tiny CNN (config 1), 1 = ResNet-50 v1.5
 * (configs 2, 3, 5), 2 = ResNet-50 v1, 3 = 3D U-Net (config 4: in_hw^3 volume, base width
 * `width` -> level widths w, 2w, 4w, 4w, input channels padded 1 -> 32), 4 = AlexNet (the
 * paper's second workload: single-tower, in_hw 227, dropout 0.5; width unused;
 * 13 maps, 62,378,344 parameters), 5 = ResNeXt-101 (3D) (the paper's third workload, SURVEY 8(f)
 * f4: input [1, D = width, H = W = in_hw, 3 -> 4 channels], 207 maps, grouped 3^3 convs), 6 = its
 * depth-50 variant ([3, 4, 6, 3] blocks; tests). which |
 * POOCH_NET_FUSE_BNRELU merges every BN-ReLU whose only consumer is a single-input 2D conv with
 * cin % 32 == 0 and stride <= 2 into that conv (POOCH_L_BNRELU_CONV; same function and
 * parameters, fewer maps: ResNet-50 105 -> 73, tiny CNN 10 -> 7). Fills up to
 * *n_layers entries of `out` (host) and sets *n_layers to the task count (call with
 * out=NULL to query). */
#define POOCH_NET_FUSE_BNRELU 16
pooch_status pooch_build_net(int32_t which, int32_t in_hw, int32_t classes, int32_t width,
                             pooch_layer_desc* out, int32_t* n_layers);

/* ---------------------------------------------------------------------------- context */
/* Creates a context for `device`. Parameters are initialised to zero; set them with
 * pooch_set_param. Returns POOCH_EUSAGE on an invalid graph (non-topological inputs,
 * unsupported shapes). */
pooch_status pooch_create(const pooch_layer_desc* layers, int32_t n_layers, const pooch_io_desc* io,
                          int32_t device, pooch_ctx** out);
void pooch_destroy(pooch_ctx* ctx);
const char* pooch_last_error(const pooch_ctx* ctx);

/* Device arena (dev_base, dev_bytes: device memory) holds EVERYTHING the library places on
 * the GPU: parameters, gradients, momentum, BN statistics, the input slot, feature maps,
 * gradient maps and workspace -- the device-memory budget of the problem statement
 * (P:L165). Host arena (host_base, host_bytes: page-locked host memory) receives swapped
 * maps. Marks any plan stale. No device work. */
pooch_status pooch_set_budget(pooch_ctx* ctx, void* dev_base, size_t dev_bytes, void* host_base,
                              size_t host_bytes);
/* Bytes of the resident part of the device arena (params, grads, momentum, stats, input
 * slot, workspace) -- the minimum budget before any feature map is placed. */
pooch_status pooch_resident_bytes(const pooch_ctx* ctx, uint64_t* out);

/* cudaStream_t handles (passed as void*): compute, swap-out (D2H), swap-in (H2D), and the
 * allreduce stream (may be NULL when world == 1). */
pooch_status pooch_set_streams(pooch_ctx* ctx, void* compute, void* d2h, void* h2d, void* comm);

/* Data parallelism: `nccl_unique_id` points at the 128-byte ncclUniqueId broadcast by the
 * caller (rank 0 creates it). The library creates its own communicator. Gradients are
 * summed across ranks and scaled by 1/world in the update. Marks the plan stale. */
pooch_status pooch_set_comm(pooch_ctx* ctx, const void* nccl_unique_id, int32_t rank, int32_t world);
/* Data parallelism over peer memory (the library's own allreduce, no NCCL): allocates this
 * rank's exchange buffer (cudaMalloc, OUTSIDE the budget arena: 64 KB of flags + one float per
 * gradient float; its size in *bytes) and writes its 64-byte cudaIpcMemHandle to handle64.
 * The caller all-gathers the handles (rank order) and passes them to pooch_set_peers, which
 * maps every other rank's buffer (cudaIpcOpenMemHandle: NVLink / NVSwitch peer memory, or the
 * same GPU when ranks share one). Each gradient bucket is then summed on the comm stream:
 * copy into the stage, barrier, rank r sums its 1/W share over all stages in rank order and
 * writes the sum into every stage, barrier, copy back -- every rank gets identical bits.
 * Gradients are scaled by 1/world in the update. Exclusive with pooch_set_comm. world <= 16.
 * A barrier whose peer never arrives traps the kernel after 120 s (a CUDA error, not a hang).
 * Marks the plan stale. Definition of the exchange: P:L12 (Sec. 1, data parallelism);
 * SURVEY 8(e). */
pooch_status pooch_peer_open(pooch_ctx* ctx, int32_t rank, int32_t world, void* handle64, uint64_t* bytes);
pooch_status pooch_set_peers(pooch_ctx* ctx, const void* handles64);
/* The communicator as NCCL reports it (ncclCommCount / ncclCommUserRank / ncclCommCuDevice):
 * ranks, this rank, CUDA device. No communicator: 1, 0, the context's device. Host only. */
pooch_status pooch_comm_info(pooch_ctx* ctx, int32_t* nranks, int32_t* rank, int32_t* cuda_device);
/* The gradient allreduce runs per bucket: reverse-layer groups of whole
 * tasks' parameters of >= 26 MB, each one contiguous float range [lo, hi) of the gradient
 * region, enqueued on the comm stream right after the backward of `close_task` (the bucket's
 * lowest-index task) and overlapping the rest of backward; SGD waits for the last one. With
 * world = 1 and a non-null id a 1-rank communicator runs the same path. Host-only query:
 * *n in = capacity of lo / hi / close_task (nullable), out = bucket count. */
pooch_status pooch_allreduce_buckets(pooch_ctx* ctx, int32_t* n, uint64_t* lo, uint64_t* hi, int32_t* close_task);

/* Precision of the tensor-core contractions (conv fwd / dgrad / wgrad, FC):
 * 1 (default) = 3xTF32 split -- each fp32 operand x is fed as x and x - tf32(x), three TF32
 * MMAs per k-step, fp32 accumulate: ~fp32-faithful, the mode the 5e-3 gradient gate holds for;
 * 0 = plain TF32 (one MMA, operands truncated to TF32 by the tensor core). Invalidates the
 * profile and the plan. */
pooch_status pooch_set_precision(pooch_ctx* ctx, int32_t precision);

/* Counter-based generator of the dropout masks (POOCH_L_FC_RELU_DROP): element i of task t's
 * output is kept iff fmix32(key ^ fmix32(i)) >= floor(p * 2^32), key = fmix32(seed ^
 * fmix32(step * 0x9E3779B9 + t)) (fmix32 = MurmurHash3's finaliser), so a recomputed forward
 * reproduces its mask. (seed, step) live in device memory; every train step advances step by
 * one after the update. Sets both; synchronises the compute stream. Valid after pooch_set_budget. */
pooch_status pooch_set_rng(pooch_ctx* ctx, uint32_t seed, uint32_t step);

/* Input slot inside the device arena: x_dev [batch, in_h, in_w, in_c] fp32 (3D networks:
 * [batch, in_d, in_h, in_w, in_c]), labels_dev [batch] int32 (POOCH_L_HEAD_CE networks: one
 * label per output voxel, [batch, d, h, w]). Valid after pooch_set_budget. */
pooch_status pooch_input_slot(pooch_ctx* ctx, float** x_dev, int32_t** labels_dev);

/* ------------------------------------------------------------------------- parameters */
pooch_status pooch_num_params(const pooch_ctx* ctx, int32_t* n);
/* name (up to 63 chars + NUL) and element count of parameter i; layout as in the header. */
pooch_status pooch_param_info(const pooch_ctx* ctx, int32_t i, char* name64, int64_t* numel);
/* which: 0 = value, 1 = gradient of the last step, 2 = momentum. Host buffers, `count`
 * floats. Synchronises the compute stream. set_param(which=0) also zeroes momentum. */
pooch_status pooch_get_param(pooch_ctx* ctx, int32_t i, int32_t which, float* host, int64_t count);
pooch_status pooch_set_param(pooch_ctx* ctx, int32_t i, int32_t which, const float* host, int64_t count);

/* ---------------------------------------------------------------------------- profile */
/* Per-task measurements of Sec. 4.2: forward / backward / recompute time,
 * swap-out / swap-in time and feature-map bytes; plus the host-link probe. Arrays are
 * context-owned and valid until the next pooch_profile / pooch_set_profile / destroy. */
typedef struct {
  int32_t n;                 /* tasks == feature maps */
  const int64_t* fwd_ns;
  const int64_t* bwd_ns;
  const int64_t* rec_ns;     /* time of the replay kernels used when the map is recomputed */
  const int64_t* d2h_ns;
  const int64_t* h2d_ns;
  const uint64_t* bytes;     /* feature-map bytes */
  int64_t tail_ns;           /* update (+ allreduce) after the last backward task */
  uint64_t resident_bytes;
  double d2h_gbs, h2d_gbs, duplex_gbs; /* probed host-link bandwidth (GB/s): one direction alone;
                                        duplex = each direction while both run (median of three,
                                        largest map that fits twice); the planner's shared-link
                                        model uses duplex / d2h and duplex / h2d (Reading 51) */
  int32_t mode;              /* how the times were measured: POOCH_PROFILE_ISOLATED or _ALL_SWAP */
  const int64_t* d2h_issue_ns; /* ALL_SWAP only (else NULL): median issue time of each map's swap-out, */
  const int64_t* h2d_issue_ns; /*   swap-in, ns after the step starts (-1: never copied)       */
  int64_t step_ns;           /* ALL_SWAP only: median measured all-swap step (0 otherwise)            */
} pooch_profile_t;

/* Profiling modes (Sec. 4.2, DESIGN.md Reading 22).
 *  ISOLATED: every task's forward, replay (recompute) and backward kernels are timed alone on
 *            scratch buffers of the dynamic region (1 warm-up + `iters` runs, median); every
 *            distinct map size is copied D2H and H2D through the pinned host arena the same way;
 *            a duplex probe copies both directions at once; the tail (weight transposes, the
 *            final bucket's allreduce at its real size, SGD) is timed likewise.
 *  ALL_SWAP: the paper's method ("all feature maps are classified into swap as the
 *            default classification"): after the isolated pass (which also provides the replay
 *            times and the numbers the all-swap plan is packed with), `iters` real steps of the
 *            all-swap plan run on the three streams after one warm-up, without the update; each
 *            task's forward / backward time and each map's D2H / H2D time become the median over
 *            those steps (under the real copy traffic), and each copy's issue time is recorded.
 *            Needs a pinned host arena holding every map and a budget in which all-swap packs.
 *  AUTO (default): ALL_SWAP when those hold, else ISOLATED (e.g. ResNet-50 at batch 2560: 214 GB
 *            of maps, more than the host's pinned memory). */
enum { POOCH_PROFILE_AUTO = 0, POOCH_PROFILE_ISOLATED = 1, POOCH_PROFILE_ALL_SWAP = 2 };
pooch_status pooch_set_profile_mode(pooch_ctx* ctx, int32_t mode);

/* Measures the profile in the context's profiling mode (above); `iters` >= 1. Parameters are NOT
 * updated; any plan is invalidated. ALL_SWAP that cannot run returns POOCH_EINFEASIBLE (AUTO
 * falls back to ISOLATED); a task whose isolated working set exceeds the budget returns
 * POOCH_EINFEASIBLE. `out` (nullable) receives context-owned arrays. */
pooch_status pooch_profile(pooch_ctx* ctx, int32_t iters, pooch_profile_t* out);
/* Replace the measured times (e.g. the element-wise max over DP ranks). Arrays of n. */
pooch_status pooch_set_profile(pooch_ctx* ctx, const int64_t* fwd_ns, const int64_t* bwd_ns,
                               const int64_t* rec_ns, const int64_t* d2h_ns, const int64_t* h2d_ns,
                               int64_t tail_ns);
/* Replace the probed host-link rates (GB/s; e.g. the most pessimistic over DP ranks, so every
 * rank plans the same). d2h / h2d: one direction alone; duplex: each direction while both run.
 * The planner's link model uses duplex / d2h and duplex / h2d (DESIGN.md Reading 51); duplex = 0
 * turns it off (independent lanes). Any plan is invalidated. EUSAGE on a negative rate, or
 * d2h / h2d <= 0 with duplex > 0. */
pooch_status pooch_set_link(pooch_ctx* ctx, double d2h_gbs, double h2d_gbs, double duplex_gbs);

/* ----------------------------------------------------------------- host-only planning */
/* A planning problem in plain arrays (host memory): the simulator's input (Sec. 4.1.2).
 * inputs / needs are CSR lists: task i consumes maps in_idx[in_ptr[i] .. in_ptr[i+1]) in
 * forward and its backward reads maps need_idx[need_ptr[i] .. need_ptr[i+1]). */
typedef struct {
  int32_t n;
  const int64_t* fwd_ns;
  const int64_t* bwd_ns;
  const int64_t* rec_ns;     /* nullable: = fwd_ns */
  const int64_t* d2h_ns;
  const int64_t* h2d_ns;
  const uint64_t* bytes;
  const int32_t* in_ptr;
  const int32_t* in_idx;
  const int32_t* need_ptr;
  const int32_t* need_idx;
  uint64_t resident_bytes;
  uint64_t budget_bytes;
  int64_t tail_ns;
  const uint8_t* is_conv;    /* nullable: 1 for convolution tasks (SuperNeurons rule only) */
  uint64_t host_budget_bytes; /* pinned host bytes for the swap class; 0 = unlimited */
  /* Shared host link (DESIGN.md Reading 51): the rate, per mille of its profiled (one-direction)
   * rate, at which a D2H / H2D copy progresses while the other copy lane is busy -- the probed
   * duplex bandwidth over the single-direction one. 0 or 1000 = independent lanes (each copy takes
   * exactly its profiled time, the plain reading of P:L165-167); valid range 1..1000. */
  int32_t duplex_d2h_permille;
  int32_t duplex_h2d_permille;
} pooch_problem;

typedef struct {
  int32_t oom;
  int64_t makespan_ns;       /* last task end, excluding tail_ns */
  uint64_t peak_bytes;
  int32_t n_events;
  /* optional outputs (nullable), arrays of n: */
  uint8_t* in_lo;            /* 1 if map in L_O */
  uint8_t* in_li;            /* 1 if map in L_I */
  int64_t* stall_ns;         /* swap-in stall charged to the map */
  /* optional event list (nullable): lane (0 COMPUTE, 1 D2H, 2 H2D), kind ('F','B','R','O','I'),
   * task id, start, end; up to events_cap entries are written. */
  int32_t events_cap;
  int32_t* ev_lane;
  int32_t* ev_kind;
  int32_t* ev_id;
  int64_t* ev_start;
  int64_t* ev_end;
} pooch_sim_result;

/* Timeline + memory simulation of one iteration under `classes` (n bytes, pooch_class;
 * 3 = zero-cost keep used for the Eq. (1) baseline). Host only, deterministic. */
pooch_status pooch_simulate(const pooch_problem* prob, const uint8_t* classes, int32_t sched,
                            pooch_sim_result* out);

typedef struct {
  int32_t li_cap;            /* max |tree| of step 1 (default 16; Reading 16) */
  int32_t threads;           /* planner threads (0 = hardware concurrency) */
  int32_t sched;             /* pooch_sched used inside the search (default EAGER) */
} pooch_search_cfg;

typedef struct {
  int64_t makespan_ns;       /* simulated iteration time incl. tail */
  uint64_t peak_bytes;       /* simulated peak device bytes (<= budget) */
  uint64_t arena_bytes;      /* packed high-water mark of the static offsets (ctx plans only) */
  int32_t n_keep, n_swap, n_recompute;  /* Table 3 counts */
  uint64_t host_bytes;       /* pinned bytes needed for the swap class */
  int64_t n_sims;
  double wall_ms;
  int32_t lo_size, li_size;  /* |L_O|, |L_I| of the all-swap timeline */
  int32_t feasible;
} pooch_plan_report;

/* Classify with `strategy` (classes_out: n bytes, host). fixed_classes only for
 * STRAT_FIXED. Returns POOCH_EINFEASIBLE when nothing fits, POOCH_EUSAGE for EXHAUSTIVE
 * with n > 12. */
pooch_status pooch_plan_problem(const pooch_problem* prob, int32_t strategy, const pooch_search_cfg* cfg,
                                const uint8_t* fixed_classes, uint8_t* classes_out,
                                pooch_plan_report* report);

/* The executor's plan refinement (DESIGN.md Reading 42; pooch_plan applies it to its best grid
 * candidates): passes over the maps trying every other class of each (the sink never
 * recompute), keeping a change when it lowers (greedy static-packing excess over `capacity`,
 * simulated makespan) lexicographically, under the simulator of Sec. 4.1.2 with the problem's
 * budget and host budget. classes_out (n) receives the result; makespan_ns (incl. tail) and
 * packs (1 = its ledger packs into capacity) nullable. POOCH_EINFEASIBLE if the start runs out
 * of memory or host arena. Host only. */
pooch_status pooch_refine_problem(const pooch_problem* prob, const uint8_t* classes, int32_t sched,
                                  uint64_t capacity, uint8_t* classes_out, int64_t* makespan_ns, int32_t* packs);

/* Static arena offsets (replaces the paper's hooked allocator): simulate `classes`,
 * replay the allocation ledger best-fit over [0, capacity). Buffer instances b in [0, 3n):
 * b = m forward instance of map m, n + m its backward-phase (swapped-in / recomputed)
 * instance, 2n + m its gradient. Outputs (host arrays of 3n, nullable except offsets):
 * byte offsets, ledger positions of allocation / free (-1 = never allocated / never freed),
 * sizes. POOCH_EINFEASIBLE on OOM or fragmentation. Host only. */
pooch_status pooch_pack_problem(const pooch_problem* prob, const uint8_t* classes, int32_t sched, uint64_t capacity,
                                uint64_t* offsets, int32_t* alloc_seq, int32_t* free_seq, uint64_t* sizes,
                                uint64_t* high_water);

/* ------------------------------------------------------------------------- execution */
/* Plans the context's network with its profile and budget, packs static arena offsets and
 * compiles the three-stream schedule. classes_out (nullable, n bytes) receives the plan. */
pooch_status pooch_plan(pooch_ctx* ctx, int32_t strategy, const pooch_search_cfg* cfg,
                        const uint8_t* fixed_classes, uint8_t* classes_out, pooch_plan_report* report);

/* One training iteration: forward, backward with swap / recompute per the plan,
 * [allreduce], momentum-SGD update with learning rate lr. The batch must already be in the
 * input slot. loss_host (nullable): if non-NULL the call synchronises and writes the mean
 * cross-entropy loss; if NULL the call only enqueues work on the caller's streams. */
pooch_status pooch_train_step(pooch_ctx* ctx, float lr, float* loss_host);

/* *graph = 1 if the last pooch_train_step ran as one captured CUDA graph launch, 0 if eagerly
 * (timing mode, POOCH_NO_GRAPH, or a capture that failed). Host only. */
pooch_status pooch_step_graph(const pooch_ctx* ctx, int32_t* graph);

/* Device address of the step's mean loss (fp32 scalar inside the arena), for callers that
 * read it back asynchronously on their own stream. */
pooch_status pooch_loss_slot(pooch_ctx* ctx, float** loss_dev);

/* Test / debug access: copies up to `bytes` of buffer instance `which` (0 = forward
 * instance, 1 = backward-phase instance, 2 = gradient) of feature map `map` as placed by the
 * current plan into `host`. Synchronises the compute stream. Contents are only meaningful
 * while the instance is live in the last step (e.g. every map under the in-core plan). */
pooch_status pooch_read_buffer(pooch_ctx* ctx, int32_t which, int32_t map, void* host, size_t bytes);

/* Instrumentation: when enabled, train_step records CUDA events around every task and copy.
 * pooch_last_timing fills per-task durations (ns, arrays of n, nullable) of the last step:
 * forward, backward, recompute (0 if none), swap-out, swap-in; and the step's total. */
pooch_status pooch_set_timing(pooch_ctx* ctx, int32_t enable);
pooch_status pooch_last_timing(pooch_ctx* ctx, int64_t* fwd_ns, int64_t* bwd_ns, int64_t* rec_ns,
                               int64_t* d2h_ns, int64_t* h2d_ns, int64_t* step_ns);

/* The measured timeline of the last instrumented step (pooch_set_timing), the executed counterpart
 * of pooch_simulate's event list: per op its lane (0 compute, 1 D2H, 2 H2D), kind ('F', 'R', 'B',
 * 'O', 'I'), task / map id and start / end in ns after the step's first event (compute ops span
 * their kernels; copies their own events). *n in = capacity of the nullable arrays, out = count. */
pooch_status pooch_last_trace(pooch_ctx* ctx, int32_t* n, int32_t* lane, int32_t* kind, int32_t* id, int64_t* start_ns,
                              int64_t* end_ns);
/* The current plan's simulated timeline (the event list its static offsets were packed from),
 * same layout as pooch_last_trace. POOCH_ENOPLAN without a plan. Host only. */
pooch_status pooch_plan_trace(pooch_ctx* ctx, int32_t* n, int32_t* lane, int32_t* kind, int32_t* id, int64_t* start_ns,
                              int64_t* end_ns);

/* Number of CUDA kernels this library launched in the last pooch_train_step (all streams;
 * copies and NCCL calls not counted). */
pooch_status pooch_kernel_launches(pooch_ctx* ctx, int64_t* per_step);

/* Kernel-family accounting of the last instrumented step: for family f (0 conv-fwd,
 * 1 conv-dgrad, 2 conv-wgrad, 3 bn-fwd, 4 bn-bwd, 5 pool, 6 fc/ce, 7 sgd, 8 swap-out,
 * 9 swap-in, 10 allreduce, 11 other, 12 compute-stream stall waiting on a copy stream, 13-15 grouped
 * conv3d fwd / dgrad / wgrad on the CUDA cores) the summed event time, launch count, algorithmic flops and
 * algorithmic DRAM bytes. */
pooch_status pooch_family_stats(pooch_ctx* ctx, int32_t family, double* time_ms, int64_t* launches,
                                double* flops, double* bytes);
/* The compute-stream segments of the last instrumented step (one per kernel launch group, in
 * enqueue order): family, event time, algorithmic flops and bytes. *n in = capacity of the
 * (nullable) arrays, out = segment count. Lets the caller put every launch against its own
 * roof (bound time = max(flops / tensor peak, bytes / HBM peak)). */
pooch_status pooch_timing_segments(pooch_ctx* ctx, int32_t* n, int32_t* family, double* time_ms, double* flops,
                                   double* bytes);

/* ---------------------------------------------------------------- kernel entry points */
/* Single convolution passes on caller device buffers, launched on `stream` (cudaStream_t).
 * Used by the parity tests; the executor calls the same launchers.
 *   fwd  : y[N,Ho,Wo,K] = conv(x[N,H,W,C], w[K,R,S,C]); stat_sum/stat_sq (nullable) receive
 *          per-M-tile column sums [pooch_op_conv_stat_tiles(d)][K].
 *   dgrad: dx[N,H,W,C] (=|+=) conv^T(dy[N,Ho,Wo,K], wt[C,R,S,K]).
 *   wgrad: dw[K,R,S,C] = sum_pixels dy x im2col(x); `ws` device workspace of ws_bytes. */
typedef struct {
  int32_t N, H, W, C, K, R, S, stride, pad;
  int32_t precision;  /* 0: TF32 operands (1 MMA per k-step); 1: 3xTF32 split, ~fp32-faithful */
  int32_t D;          /* 0: 2D. > 0: 3D conv3d over x[1,D,H,W,C] (N must be 1), kernel R^3,
                         weights [K,R,R,R,C]; requires C, K multiples of 32 (TMA-fed kernels) */
  int32_t C1;         /* 0: one input. > 0: the input is the channel concatenation of two
                         tensors x0 [..,C1] and x1 [..,C-C1] (the *2 entry points); C1 % 32 == 0 */
  int32_t groups;     /* 0 / 1: dense. > 1: grouped 3D conv (ResNeXt-101 (3D), SURVEY 8(f) f4;
                         definition: oracle layers.gconv3d_fwd, the aggregated transformation of
                         P:L386's ResNeXt): D > 0, C == K, C / groups in {4, 8, 16, 32}, K % 32 == 0,
                         R == S in {1, 3}, one stride (1 or 2) on all three axes; weights
                         [K][R][R][R][C/groups], and dgrad
                         reads that same (untransposed) layout as `wt`. FP32 on the CUDA cores. */
  int32_t stride_d;   /* 3D: stride along depth; 0 = `stride` (ResNeXt-101 (3D)'s stem: 1, 2, 2) */
} pooch_conv_desc;

pooch_status pooch_op_conv_fwd(const pooch_conv_desc* d, const float* x, const float* w, float* y,
                               float* stat_sum, float* stat_sq, void* stream);
pooch_status pooch_op_conv_dgrad(const pooch_conv_desc* d, const float* dy, const float* wt, float* dx,
                                 int32_t accumulate, void* stream);
pooch_status pooch_op_conv_wgrad(const pooch_conv_desc* d, const float* x, const float* dy, float* dw,
                                 float* ws, size_t ws_bytes, void* stream);
size_t pooch_op_conv_wgrad_ws_bytes(const pooch_conv_desc* d);
/* Two-source variants (d->C1 > 0): the convolution's input is concat_c(x0, x1), read in place
 * (never materialised); dgrad writes (or accumulates into, per destination) dx0 and dx1. */
pooch_status pooch_op_conv_fwd2(const pooch_conv_desc* d, const float* x0, const float* x1, const float* w, float* y,
                                float* stat_sum, float* stat_sq, void* stream);
pooch_status pooch_op_conv_dgrad2(const pooch_conv_desc* d, const float* dy, const float* wt, float* dx0, float* dx1,
                                  int32_t accumulate0, int32_t accumulate1, void* stream);
pooch_status pooch_op_conv_wgrad2(const pooch_conv_desc* d, const float* x0, const float* x1, const float* dy,
                                  float* dw, float* ws, size_t ws_bytes, void* stream);
/* BN-ReLU applied to the activation operand on load (the POOCH_L_BNRELU_CONV
 * kernels): the convolution's input is relu(scale[c] * x + shift[c]) (scale / shift: device [C],
 * the BN's gamma * invstd and beta - mean * gamma * invstd), zero padding stays zero. 2D, one
 * source, C % 32 == 0, stride <= 2 (TMA-fed kernels), else POOCH_EUSAGE. */
pooch_status pooch_op_conv_fwd_bnrelu(const pooch_conv_desc* d, const float* x, const float* scale,
                                      const float* shift, const float* w, float* y, float* stat_sum,
                                      float* stat_sq, void* stream);
pooch_status pooch_op_conv_wgrad_bnrelu(const pooch_conv_desc* d, const float* x, const float* scale,
                                        const float* shift, const float* dy, float* dw, float* ws,
                                        size_t ws_bytes, void* stream);
/* Number of M-tiles (rows of the partial-sum arrays) of pooch_op_conv_fwd for `d`. */
int64_t pooch_op_conv_stat_tiles(const pooch_conv_desc* d);
/* 2D max-pool (k x k window, stride s, padding p with -inf; Sec. 2.1 layer math, DESIGN.md
 * Reading 25) on NHWC device buffers, launched on `stream`. fwd: y[N,Ho,Wo,C]. bwd: gx[N,H,W,C] =
 * the gradient routed to the FIRST maximum (row-major window order) of every window, recomputed
 * from x; `arg_ws` is a device workspace of N*Ho*Wo*C bytes. C % 4 == 0, H*W*C < 2^31, else
 * POOCH_EUSAGE. Ho = (H + 2p - k)/s + 1 (likewise Wo). Used by the parity tests; the executor
 * calls the same launchers. */
pooch_status pooch_op_maxpool2d_fwd(const float* x, float* y, int32_t N, int32_t H, int32_t W, int32_t C, int32_t k,
                                    int32_t s, int32_t p, void* stream);
pooch_status pooch_op_maxpool2d_bwd(const float* x, const float* gy, float* gx, void* arg_ws, int32_t N, int32_t H,
                                    int32_t W, int32_t C, int32_t k, int32_t s, int32_t p, void* stream);
/* Training-mode BN + ReLU passes the executor runs after a convolution (Sec. 2.1 layer math; the
 * 3D U-Net's conv3d -> BN -> ReLU -> max-pool chain), on NDHWC / NHWC device buffers of `rows`
 * pixels x C channels (C % 4 == 0; rows * C may exceed 2^31), launched on `stream`:
 *   bn_finalize : per-channel mean, invstd = 1/sqrt(var + 1e-5), scale = gamma * invstd,
 *                 shift = beta - mean * scale (each [C]) from the conv forward's per-M-tile column
 *                 sums tile_sum / tile_sq [tiles][C] (pooch_op_conv_fwd's stat_sum / stat_sq) over
 *                 `count` pixels, reduced in a fixed order in fp64; ws: pooch_op_bn_ws_bytes(C) B.
 *   bn_relu_fwd : y = relu(fma(x, scale, shift)).
 *   bn_relu_bwd : dz = gy * [relu input > 0] (recomputed from x, scale, shift exactly as the forward);
 *                 dbeta = sum dz, dgamma = sum dz * xhat (per channel, fixed order);
 *                 gx = gamma * invstd * (dz - dbeta / rows - xhat * dgamma / rows); ws as above.
 * 3D max-pool, 2x2x2 windows, stride 2, no padding, over x [D][H][W][C] (batch 1):
 *   maxpool3d_fwd : y [D/2][H/2][W/2][C];  maxpool3d_bwd : gx (=|+=) the gradient routed to the FIRST
 *                 maximum of every window in (d, h, w) row-major order (Reading 25), argmax from x.
 * POOCH_EUSAGE on null pointers or bad shapes. Used by the parity tests. */
size_t pooch_op_bn_ws_bytes(int32_t C);
/* AlexNet's local response normalisation over the C (<= 1024) channels of `pixels` NHWC pixels:
 * lrn_fwd y = x * s^-0.75, s = 2 + 1e-4 / 5 * sum_{|c'-c| <= 2} x_c'^2; lrn_bwd gx = its adjoint
 * applied to gy (written, not accumulated). */
pooch_status pooch_op_lrn_fwd(const float* x, float* y, int64_t pixels, int32_t C, void* stream);
pooch_status pooch_op_lrn_bwd(const float* x, const float* gy, float* gx, int64_t pixels, int32_t C, void* stream);
pooch_status pooch_op_bn_finalize(const float* tile_sum, const float* tile_sq, int32_t tiles, int32_t C, int64_t count,
                                  const float* gamma, const float* beta, float* mean, float* invstd, float* scale,
                                  float* shift, void* ws, void* stream);
pooch_status pooch_op_bn_relu_fwd(const float* x, const float* scale, const float* shift, float* y, int64_t rows,
                                  int32_t C, void* stream);
pooch_status pooch_op_bn_relu_bwd(const float* x, const float* gy, const float* scale, const float* shift,
                                  const float* mean, const float* invstd, const float* gamma, float* dgamma,
                                  float* dbeta, float* gx, int64_t rows, int32_t C, void* ws, void* stream);
pooch_status pooch_op_maxpool3d_fwd(const float* x, float* y, int32_t D, int32_t H, int32_t W, int32_t C, void* stream);
pooch_status pooch_op_maxpool3d_bwd(const float* x, const float* gy, float* gx, int32_t D, int32_t H, int32_t W,
                                    int32_t C, int32_t accumulate, void* stream);
/* 3D max-pool with any k / s / p (-inf padding; ResNeXt-101 (3D)'s 3^3 / 2 pad 1):
 * y [Do][Ho][Wo][C], Do = (D + 2p - k)/s + 1; bwd gx (=|+=) the gradient routed to the first
 * maximum of every window in (d, h, w) row-major order (Reading 25), gathered from the input side
 * (overlapping windows add in output order); arg_ws: device workspace of Do*Ho*Wo*C bytes.
 * k2 s2 p0 runs the tiling kernels above (arg_ws unused). C % 4 == 0, 1 <= k <= 6, p < k. */
pooch_status pooch_op_maxpool3d_fwd_k(const float* x, float* y, int32_t D, int32_t H, int32_t W, int32_t C, int32_t k,
                                      int32_t s, int32_t p, void* stream);
pooch_status pooch_op_maxpool3d_bwd_k(const float* x, const float* gy, float* gx, void* arg_ws, int32_t D, int32_t H,
                                      int32_t W, int32_t C, int32_t k, int32_t s, int32_t p, int32_t accumulate,
                                      void* stream);
/* ---------------------------------------------------------------- intra-layer division */
/* ooc_cuDNN-style division of a single layer whose maps exceed the device (P:L495,
 * Sec. 6: "ooc_cuDNN performs data-swapping after dividing each computation and data ... supports
 * NNs where memory consumption of a single layer exceeds the GPU memory capacity"). Tensors are
 * HOST-resident (pinned, NDHWC, batch 1); the layer runs in chunks of depth rows through the
 * caller's device workspace `ws` of ws_bytes (the chunk size is the largest that fits two buffer
 * sets), the copies of one chunk overlapping the kernels of the next on three streams (`streams`:
 * compute, H2D, D2H cudaStream_t). A convolution chunk loads its input rows plus the halo rows
 * (zero rows at the volume's faces) and runs the undivided kernels on the slab, padded in H / W
 * only, so conv fwd / dgrad outputs equal the undivided launch bit for bit; BN statistics and
 * wgrad partials are summed over chunks in chunk order (fp64 / fp32). Synchronous: returns when
 * done; *info (nullable) gets the chunking, the device time and the bytes moved. POOCH_EINFEASIBLE
 * when one row does not fit ws; POOCH_EUSAGE for unsupported shapes (3D dense single-source
 * convs, one stride on all axes, kernel >= stride). */
typedef struct {
  int32_t chunks, rows_per_chunk;
  double ms;
  uint64_t h2d_bytes, d2h_bytes;
} pooch_div_info;
/* y = conv3d(x, w) (x [D][H][W][C] host, w device KTRSC, y [Do][Ho][Wo][K] host). With `stats`
 * (device [4K]: mean, invstd, scale, shift) the training-mode BN statistics of y are computed
 * (bn_finalize's formula, eps 1e-5) for gamma / beta (device [K]). */
pooch_status pooch_div_conv3d_fwd(const pooch_conv_desc* d, const float* x_host, const float* w_dev, float* y_host,
                                  const float* gamma, const float* beta, float* stats, void* ws, size_t ws_bytes,
                                  void* const* streams, pooch_div_info* info);
/* y = relu(scale[c] c + shift[c]) over rows x row_floats (row_floats = H W C) host floats. */
pooch_status pooch_div_bn_relu_fwd(const float* c_host, const float* stats, float* y_host, int64_t rows,
                                   int64_t row_floats, int32_t C, void* ws, size_t ws_bytes, void* const* streams,
                                   pooch_div_info* info);
/* BN-ReLU backward in two passes over the chunks: dbeta = sum dz, dgamma = sum dz xhat (device [C]),
 * gx = gamma invstd (dz - dbeta / M - xhat dgamma / M), dz = gy [relu input > 0]. */
pooch_status pooch_div_bn_relu_bwd(const float* c_host, const float* gy_host, const float* stats, const float* gamma,
                                   float* dgamma, float* dbeta, float* gx_host, int64_t rows, int64_t row_floats,
                                   int32_t C, void* ws, size_t ws_bytes, void* const* streams, pooch_div_info* info);
/* gx = conv3d^T(gy, wt) (wt device [C][T][R][S][K], as pooch_op_conv_dgrad), host in / out. */
pooch_status pooch_div_conv3d_dgrad(const pooch_conv_desc* d, const float* gy_host, const float* wt_dev,
                                    float* gx_host, void* ws, size_t ws_bytes, void* const* streams,
                                    pooch_div_info* info);
/* dw (device KTRSC) = sum over chunks of the chunk's wgrad (x, gy host). */
pooch_status pooch_div_conv3d_wgrad(const pooch_conv_desc* d, const float* x_host, const float* gy_host,
                                    float* dw_dev, void* ws, size_t ws_bytes, void* const* streams,
                                    pooch_div_info* info);

/* D[split][M][N] = A * B^T on the tensor-core core, A [M][K] and B [N][K] row-major (K-major);
 * a_mn = 2 selects the 3xTF32 path, other non-zero a_mn / b_mn (MN-major operands) return
 * POOCH_EUSAGE; bn in {64,128,256} (64/128 for 3xTF32); splits >= 1. Unit test only. */
pooch_status pooch_op_gemm_test(const float* A, const float* B, float* D, int32_t M, int32_t N, int32_t K,
                                int32_t a_mn, int32_t b_mn, int32_t bn, int32_t splits, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* POOCH_H */
