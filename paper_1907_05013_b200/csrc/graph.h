// graph.h -- task graph of the network and the planning problem derived from it.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/pooch.h"

namespace pooch {

// One fused executor task; its output is one feature map. Shapes are per image.
struct Task {
  int kind;            // pooch_layer_kind
  int in0, in1;        // producer ids, -1 = network input / unused
  int cin, cout, hout, wout, k, stride, pad;
  int hin, win;        // derived: input spatial dims (conv / pool)
  int din, dout;       // 3D networks: input / output depth (0 in 2D networks)
  int groups = 1;      // grouped conv (ResNeXt-101 (3D)); 1 = dense
  int stride_d = 0;    // 3D conv: depth stride (0 = stride)
  std::string name;
  std::vector<int> inputs;  // map inputs (ids >= 0)
  std::vector<int> needs;   // maps bwd(task) reads
  std::vector<int> consumers;
  uint64_t map_bytes;       // per batch
};

struct Graph {
  std::vector<Task> t;
  pooch_io_desc io;
  int n() const { return (int)t.size(); }
};

// Validates and derives inputs / needs / consumers / bytes; returns false + message on error.
bool build_graph(const pooch_layer_desc* layers, int n, const pooch_io_desc& io, Graph& g, std::string& err);

// The planning problem in owned arrays (mirrors pooch_problem).
struct Problem {
  int n = 0;
  std::vector<int64_t> fwd, bwd, rec, d2h, h2d;
  std::vector<uint64_t> bytes;
  std::vector<std::vector<int>> inputs, needs;
  std::vector<uint8_t> is_conv;
  uint64_t resident = 0, budget = 0;
  uint64_t host_budget = 0;  // 0: unlimited
  // shared host link (Reading 51): per-mille rate of a D2H / H2D copy while the other copy lane is
  // busy (probed duplex / single-direction bandwidth); 1000 (or 0) = independent lanes
  int duplex_d2h = 1000, duplex_h2d = 1000;
  int64_t tail = 0;
};

bool problem_from_c(const pooch_problem& p, Problem& out, std::string& err);

}  // namespace pooch
