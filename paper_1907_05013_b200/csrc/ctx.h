// ctx.h -- the pooch_ctx: resident layout, plan, packed offsets and compiled three-stream
// schedule of the out-of-core executor.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/pooch.h"
#include "conv.h"
#include "graph.h"
#include "sim.h"

namespace pooch {

enum Family {
  FAM_CONV_FWD = 0, FAM_CONV_DGRAD, FAM_CONV_WGRAD, FAM_BN_FWD, FAM_BN_BWD, FAM_POOL, FAM_FC_CE, FAM_SGD,
  FAM_SWAP_OUT, FAM_SWAP_IN, FAM_ALLREDUCE, FAM_OTHER, FAM_STALL,
  FAM_GCONV_FWD, FAM_GCONV_DGRAD, FAM_GCONV_WGRAD,  // grouped conv3d on the CUDA cores (ALU roof)
  FAM_COUNT
};

struct ParamT {
  std::string name;
  int task;
  int64_t numel;
  size_t off;  // float offset inside the param region
};

// Per task resident pointers / derived geometry
struct TaskRt {
  ConvGeom geom{};      // conv / fc
  bool is_conv = false; // conv or fc (uses the igemm)
  int w = -1, b = -1;   // param indices (conv/fc weight, fc bias)
  int g1 = -1, b1 = -1, g2 = -1, b2 = -1;  // BN params: (gamma, beta) of BN(in0) [and BN(in1)]
  size_t wt_off = 0;    // float offset of the transposed weight in the wt region
  // BN statistics of this task's output (conv outputs feeding a BN): floats offset, 4*C
  size_t stat_off = 0;
  bool has_stats = false;
  int bn_gamma = -1, bn_beta = -1;  // params of the BN consuming this conv output
  int64_t rows = 0;     // N*H*W of the output
  int cpad = 0;         // FC: padded classes
  double flops = 0;     // per pass (fwd == dgrad == wgrad for convs)
  // 3D stem with depth stride 1 reading the network input (ResNeXt-101 (3D)'s 7^3 conv): run as a
  // 2D conv over the Do depth slices of the input's depth-im2col X'[od][h][w][u*C + c] =
  // x[od+u-p][h][w][c] (k*C <= 32 channels, padded to 32), geom holds that 2D geometry, the wt
  // region holds the weight re-laid [K][v][t][u*C + c]; fold_c = C, fold_k = k
  bool fold = false;
  int fold_c = 0, fold_k = 0;
};

// One host-enqueued operation of the compiled schedule.
struct Op {
  int lane;   // 0 compute, 1 d2h, 2 h2d
  char kind;  // 'F','R','B','O','I'
  int id;
  std::vector<int> waits;  // op indices on other lanes whose completion event must be waited
  bool record = false;     // another lane waits on this op's completion
  bool record_start = false;  // another lane waits on this op's start (naive / SN swap-in triggers)
  std::vector<int> start_waits;  // compute ops whose START must precede this op
  std::vector<int> frees;        // POOCH_DEBUG_POISON: buffer instances this op frees (NaN-filled after it)
};

struct pooch_ctx_impl;

}  // namespace pooch

struct pooch_ctx {
  pooch::Graph g;
  int device = 0;
  std::string err;
  // arenas
  char* dev = nullptr;
  size_t dev_bytes = 0;
  char* host = nullptr;
  size_t host_bytes = 0;
  // streams
  cudaStream_t s[4] = {nullptr, nullptr, nullptr, nullptr};  // compute, d2h, h2d, comm
  bool own_streams = false;
  // resident layout
  std::vector<pooch::ParamT> params;
  int64_t param_floats = 0;
  std::vector<pooch::TaskRt> rt;
  size_t off_w = 0, off_g = 0, off_v = 0, off_wt = 0, off_stats = 0, off_tile = 0, off_fin = 0, off_bnws = 0,
         off_wgws = 0, off_mparg = 0, off_x = 0, off_lab = 0, off_lossrows = 0, off_loss = 0, off_dz = 0,
         off_cews = 0, off_rng = 0, off_xs = 0, off_w2g = 0;  // off_cews: CE two-stage reduction scratch; off_rng: dropout {seed, step}
  size_t xs_bytes = 0, w2g_bytes = 0;  // folded stem: depth-im2col input X', wgrad scratch dW'
  size_t wt_floats = 0, stats_floats = 0, tile_bytes = 0, fin_bytes = 0, bnws_bytes = 0, wgws_bytes = 0,
         mparg_bytes = 0;
  size_t resident_end = 0;
  bool budget_set = false;
  // profile
  std::vector<int64_t> fwd_ns, bwd_ns, rec_ns, d2h_ns, h2d_ns;
  std::vector<uint64_t> map_bytes;
  int64_t tail_ns = 0;
  double d2h_gbs = 0, h2d_gbs = 0, duplex_gbs = 0;
  bool have_profile = false;
  int profile_mode = 0;        // requested: POOCH_PROFILE_AUTO / _ISOLATED / _ALL_SWAP
  int profile_mode_used = 0;   // what the last pooch_profile measured (ISOLATED or ALL_SWAP)
  std::vector<int64_t> prof_d2h_issue, prof_h2d_issue;  // all-swap mode: per-map copy issue (ns from step start)
  int64_t prof_step_ns = 0;    // all-swap mode: median measured step time of the profiling iterations
  // plan
  std::vector<uint8_t> cls;
  bool have_plan = false;
  std::vector<size_t> buf_off;   // 3n buffer instances: fwd, bwd, grad (byte offset in dev)
  std::vector<size_t> host_off;  // per map, swap class only
  uint64_t arena_high = 0;
  uint64_t plan_budget = 0;      // simulator budget of the chosen candidate (<= arena capacity)
  bool refined = false, plan_refined = false;  // the plan came out of the local refinement (Reading 42)
  // the step captured as one CUDA graph (re-captured when the plan, streams or lr change)
  uint64_t plan_version = 0, graph_version = ~0ull;
  float graph_lr = 0.f;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  bool graphs_off = false;
  bool last_step_graph = false;  // the last pooch_train_step ran as a CUDA graph launch
  bool poison = false;           // POOCH_DEBUG_POISON at the last compile
  cudaEvent_t ev_join[3] = {nullptr, nullptr, nullptr};
  std::vector<pooch::Op> ops;
  std::vector<pooch::ProgTask> program;
  std::vector<pooch::SimEvent> plan_events;  // the adopted plan's simulated timeline
  std::vector<int> first_writer;  // per map: task whose bwd writes (not accumulates) its gradient
  // events
  std::vector<cudaEvent_t> ev;    // one per op (sync events)
  std::vector<cudaEvent_t> ev_start;  // start events (only for ops with record_start)
  int sched = 0;                  // swap-in schedule of the current plan
  // timing
  bool timing = false;
  std::vector<cudaEvent_t> tev;   // timing events
  std::vector<std::pair<int, int>> tseg;  // (event index start, family), per segment
  std::vector<double> seg_flops, seg_bytes;
  std::vector<int> seg_task, seg_kind;  // task id and 'F','R','B','O','I','U'
  std::vector<double> seg_ms_last;      // per-segment event time of the last instrumented step
  int t_used = 0;
  double fam_ms[pooch::FAM_COUNT] = {0};
  int64_t fam_launch[pooch::FAM_COUNT] = {0};
  double fam_flops[pooch::FAM_COUNT] = {0}, fam_bytes[pooch::FAM_COUNT] = {0};
  std::vector<int64_t> last_fwd, last_bwd, last_rec, last_d2h, last_h2d;
  std::vector<int64_t> last_d2h_issue, last_h2d_issue;  // copy start, ns after the step's first event
  struct TraceEv {
    int lane;
    char kind;
    int id;
    int64_t start, end;
  };
  std::vector<TraceEv> trace;  // measured timeline of the last instrumented step
  int64_t last_step_ns = 0;
  // dp
  void* nccl = nullptr;
  int rank = 0, world = 1;
  // peer-memory allreduce (peer.cu): own IPC-exported exchange buffer, every rank's mapped base
  void* peer_own = nullptr;
  std::vector<void*> peer_base;
  size_t peer_floats = 0;
  int sm_count = 148;
  // gradient allreduce buckets (reverse-layer order, ~26 MB): float range of the gradient
  // region and the task whose backward completes it; events compute -> comm and comm -> update
  struct Bucket {
    size_t lo, hi;
    int close_task;
  };
  std::vector<Bucket> buckets;
  std::vector<int> bucket_at;            // task -> bucket index closed by its backward, or -1
  std::vector<cudaEvent_t> ev_bucket;
  cudaEvent_t ev_comm_done = nullptr;
  cudaStream_t own_comm = nullptr;
  int64_t step_count = 0;
  int64_t last_launches = 0;
  int precision = 1;  // contractions: 0 TF32, 1 3xTF32 (default; DESIGN.md Reading 27)
  bool has_dropout = false;  // an FC_RELU_DROP task with p > 0: the step counter advances per step
};

namespace pooch {
// peer.cu: allreduce (sum) of src[0, hi - lo) through stage range [lo, hi) of the exchange
// buffers; `slot` numbers the barrier pair (buckets 0..n-1, the profile tail n)
pooch_status peer_allreduce(pooch_ctx* c, float* src, size_t lo, size_t hi, int slot, cudaStream_t st);
void peer_close(pooch_ctx* c);
int peer_max_slots();
// executor.cpp: buckets + events for the comm stream
void peer_setup_buckets(pooch_ctx* c);
// the step exchanges gradients (NCCL communicator or peer-memory buffers)
inline bool has_comm(const pooch_ctx* c) { return c->nccl != nullptr || !c->peer_base.empty(); }
}  // namespace pooch
