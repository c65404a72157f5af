// graph.cpp -- network builders (tiny CNN, ResNet-50, 3D U-Net, AlexNet) and task-graph derivation.
//
// Feature maps are the task outputs retained for backward (Sec. 2.1; P:L160,
// Sec. 4.1.1). For ResNet-50 the census is 53 conv + 49 BN(+add)+ReLU + maxpool + avgpool
// + FC = 105 maps, the row total of Table 3.
#include <algorithm>
#include <cstring>

#include "common.h"
#include "graph.h"

namespace pooch {

namespace {

struct Builder {
  std::vector<pooch_layer_desc> out;
  int add(int kind, int in0, int in1, int cin, int cout, int h, int w, int k, int s, int p, const std::string& nm,
          int dout = 0, int groups = 0, int stride_d = 0) {
    pooch_layer_desc d{};
    d.kind = kind; d.in0 = in0; d.in1 = in1; d.cin = cin; d.cout = cout; d.hout = h; d.wout = w;
    d.k = k; d.stride = s; d.pad = p; d.dout = dout; d.groups = groups; d.stride_d = stride_d;
    std::snprintf(d.name, sizeof(d.name), "%s", nm.c_str());
    out.push_back(d);
    return (int)out.size() - 1;
  }
};

int co(int h, int k, int s, int p) { return (h + 2 * p - k) / s + 1; }

void tiny(Builder& b, int hw, int classes, int width) {
  int src = -1, cin = 4;  // input channels padded 3 -> 4
  for (int l = 0; l < 4; ++l) {
    int c = b.add(POOCH_L_CONV, src, -1, cin, width, hw, hw, 3, 1, 1, "conv" + std::to_string(l));
    src = b.add(POOCH_L_BNRELU, c, -1, width, width, hw, hw, 0, 1, 0, "bn" + std::to_string(l));
    cin = width;
  }
  int h2 = hw / 2;
  int p = b.add(POOCH_L_MAXPOOL, src, -1, width, width, h2, h2, 2, 2, 0, "maxpool");
  b.add(POOCH_L_FC_CE, p, -1, width * h2 * h2, classes, 1, 1, 0, 1, 0, "fc");
}

void resnet50(Builder& b, int in_hw, int classes, bool v15) {
  int hw = co(in_hw, 7, 2, 3);
  int c = b.add(POOCH_L_CONV, -1, -1, 4, 64, hw, hw, 7, 2, 3, "conv1");
  int x = b.add(POOCH_L_BNRELU, c, -1, 64, 64, hw, hw, 0, 1, 0, "bn1");
  hw = co(hw, 3, 2, 1);
  x = b.add(POOCH_L_MAXPOOL, x, -1, 64, 64, hw, hw, 3, 2, 1, "maxpool");
  int cin = 64;
  const int nblocks[4] = {3, 4, 6, 3}, mids[4] = {64, 128, 256, 512};
  for (int si = 0; si < 4; ++si) {
    int mid = mids[si], out = 4 * mid;
    for (int bi = 0; bi < nblocks[si]; ++bi) {
      int s = (bi == 0 && si > 0) ? 2 : 1;
      std::string pre = "layer" + std::to_string(si + 1) + "." + std::to_string(bi);
      int s1 = v15 ? 1 : s, s2 = v15 ? s : 1;
      int hw1 = co(hw, 1, s1, 0);
      int c1 = b.add(POOCH_L_CONV, x, -1, cin, mid, hw1, hw1, 1, s1, 0, pre + ".conv1");
      int y1 = b.add(POOCH_L_BNRELU, c1, -1, mid, mid, hw1, hw1, 0, 1, 0, pre + ".bn1");
      int hw2 = co(hw1, 3, s2, 1);
      int c2 = b.add(POOCH_L_CONV, y1, -1, mid, mid, hw2, hw2, 3, s2, 1, pre + ".conv2");
      int y2 = b.add(POOCH_L_BNRELU, c2, -1, mid, mid, hw2, hw2, 0, 1, 0, pre + ".bn2");
      int c3 = b.add(POOCH_L_CONV, y2, -1, mid, out, hw2, hw2, 1, 1, 0, pre + ".conv3");
      if (bi == 0) {
        int p = b.add(POOCH_L_CONV, x, -1, cin, out, hw2, hw2, 1, s, 0, pre + ".downsample");
        x = b.add(POOCH_L_TAIL_PROJ, c3, p, out, out, hw2, hw2, 0, 1, 0, pre + ".tail");
      } else {
        x = b.add(POOCH_L_TAIL_ID, c3, x, out, out, hw2, hw2, 0, 1, 0, pre + ".tail");
      }
      hw = hw2;
      cin = out;
    }
  }
  int a = b.add(POOCH_L_AVGPOOL, x, -1, cin, cin, 1, 1, 0, 1, 0, "avgpool");
  b.add(POOCH_L_FC_CE, a, -1, cin, classes, 1, 1, 0, 1, 0, "fc");
}

// AlexNet (oracle nets.alexnet, same tasks): conv+bias+ReLU, LRN, 3/2 max-pool,
// FC+ReLU+dropout, FC+CE; input 227x227, channels padded 3 -> 4.
void alexnet(Builder& b, int in_hw, int classes) {
  int h = co(in_hw, 11, 4, 0);
  int x = b.add(POOCH_L_CONV_RELU, -1, -1, 4, 96, h, h, 11, 4, 0, "conv1");
  x = b.add(POOCH_L_LRN, x, -1, 96, 96, h, h, 0, 1, 0, "lrn1");
  h = co(h, 3, 2, 0);
  x = b.add(POOCH_L_MAXPOOL, x, -1, 96, 96, h, h, 3, 2, 0, "pool1");
  x = b.add(POOCH_L_CONV_RELU, x, -1, 96, 256, h, h, 5, 1, 2, "conv2");
  x = b.add(POOCH_L_LRN, x, -1, 256, 256, h, h, 0, 1, 0, "lrn2");
  h = co(h, 3, 2, 0);
  x = b.add(POOCH_L_MAXPOOL, x, -1, 256, 256, h, h, 3, 2, 0, "pool2");
  x = b.add(POOCH_L_CONV_RELU, x, -1, 256, 384, h, h, 3, 1, 1, "conv3");
  x = b.add(POOCH_L_CONV_RELU, x, -1, 384, 384, h, h, 3, 1, 1, "conv4");
  x = b.add(POOCH_L_CONV_RELU, x, -1, 384, 256, h, h, 3, 1, 1, "conv5");
  h = co(h, 3, 2, 0);
  x = b.add(POOCH_L_MAXPOOL, x, -1, 256, 256, h, h, 3, 2, 0, "pool5");
  x = b.add(POOCH_L_FC_RELU_DROP, x, -1, 256 * h * h, 4096, 1, 1, 50, 1, 0, "fc6");
  x = b.add(POOCH_L_FC_RELU_DROP, x, -1, 4096, 4096, 1, 1, 50, 1, 0, "fc7");
  b.add(POOCH_L_FC_CE, x, -1, 4096, classes, 1, 1, 0, 1, 0, "fc8");
}

// 3D U-Net of BASELINE config 4: 4 levels of widths w, 2w, 4w, 4w, each
// 2 x [conv3d 3^3 -> BN -> ReLU]; 2^3 max-pool; 4w bottleneck; decoder: k2 s2 transposed conv
// to the level width, then the first conv reads [up, skip] as two sources; 1^3 head + voxel CE.
void unet3d(Builder& b, int e, int classes, int w) {
  const int widths[4] = {w, 2 * w, 4 * w, 4 * w};
  int src = -1, c = 32;  // input channels padded 1 -> 32 (every 3D conv is TMA-fed)
  int skip[4], skw[4], ske[4];
  auto block = [&](const std::string& pre, int x0, int x1, int cin, int cw, int ee) {
    int c1 = b.add(POOCH_L_CONV, x0, x1, cin, cw, ee, ee, 3, 1, 1, pre + ".conv1", ee);
    int y1 = b.add(POOCH_L_BNRELU, c1, -1, cw, cw, ee, ee, 0, 1, 0, pre + ".bn1", ee);
    int c2 = b.add(POOCH_L_CONV, y1, -1, cw, cw, ee, ee, 3, 1, 1, pre + ".conv2", ee);
    return b.add(POOCH_L_BNRELU, c2, -1, cw, cw, ee, ee, 0, 1, 0, pre + ".bn2", ee);
  };
  for (int lv = 0; lv < 4; ++lv) {
    int y = block("enc" + std::to_string(lv + 1), src, -1, c, widths[lv], e);
    skip[lv] = y; skw[lv] = widths[lv]; ske[lv] = e;
    e /= 2;
    src = b.add(POOCH_L_MAXPOOL, y, -1, widths[lv], widths[lv], e, e, 2, 2, 0, "pool" + std::to_string(lv + 1), e);
    c = widths[lv];
  }
  src = block("mid", src, -1, c, widths[3], e);
  c = widths[3];
  for (int lv = 3; lv >= 0; --lv) {
    e = ske[lv];
    int u = b.add(POOCH_L_UPCONV, src, -1, c, skw[lv], e, e, 2, 2, 0, "up" + std::to_string(lv + 1), e);
    src = block("dec" + std::to_string(lv + 1), u, skip[lv], 2 * skw[lv], skw[lv], e);
    c = skw[lv];
  }
  b.add(POOCH_L_HEAD_CE, src, -1, c, classes, e, e, 1, 1, 0, "head", e);
}

// ResNeXt-101 (3D) (oracle nets.resnext3d, same tasks): conv 7^3 stride
// (1, 2, 2) pad 3 -> BN-ReLU -> max-pool 3^3 / 2 pad 1; [3, 4, 23, 3] bottlenecks of widths 128 /
// 256 / 512 / 1024 with a grouped (32) 3^3 conv, 2x expansion, projection shortcut in each stage's
// first block; global average pool; FC. Input [1, D, H, W, 3 -> 4 channels]; the stem runs
// depth-folded (executor TaskRt::fold: 7 depth taps x 4 channels as 28 -> 32 channels of a 2D conv).
void resnext3d(Builder& b, int d, int hw, int classes, int depth) {
  const int n101[4] = {3, 4, 23, 3}, n50[4] = {3, 4, 6, 3};
  const int* nb = depth == 50 ? n50 : n101;
  const int mids[4] = {128, 256, 512, 1024};
  int e = d, h = co(hw, 7, 2, 3);
  int c = b.add(POOCH_L_CONV, -1, -1, 4, 64, h, h, 7, 2, 3, "conv1", e, 0, 1);
  int x = b.add(POOCH_L_BNRELU, c, -1, 64, 64, h, h, 0, 1, 0, "bn1", e);
  e = co(e, 3, 2, 1);
  h = co(h, 3, 2, 1);
  x = b.add(POOCH_L_MAXPOOL, x, -1, 64, 64, h, h, 3, 2, 1, "maxpool", e);
  int cin = 64;
  for (int si = 0; si < 4; ++si) {
    const int mid = mids[si], out = 2 * mid;
    for (int bi = 0; bi < nb[si]; ++bi) {
      const int s = (bi == 0 && si > 0) ? 2 : 1;
      const std::string pre = "layer" + std::to_string(si + 1) + "." + std::to_string(bi);
      int c1 = b.add(POOCH_L_CONV, x, -1, cin, mid, h, h, 1, 1, 0, pre + ".conv1", e);
      int y1 = b.add(POOCH_L_BNRELU, c1, -1, mid, mid, h, h, 0, 1, 0, pre + ".bn1", e);
      const int e2 = co(e, 3, s, 1), h2 = co(h, 3, s, 1);
      int c2 = b.add(POOCH_L_CONV, y1, -1, mid, mid, h2, h2, 3, s, 1, pre + ".conv2", e2, 32);
      int y2 = b.add(POOCH_L_BNRELU, c2, -1, mid, mid, h2, h2, 0, 1, 0, pre + ".bn2", e2);
      int c3 = b.add(POOCH_L_CONV, y2, -1, mid, out, h2, h2, 1, 1, 0, pre + ".conv3", e2);
      if (bi == 0) {
        int p = b.add(POOCH_L_CONV, x, -1, cin, out, h2, h2, 1, s, 0, pre + ".downsample", e2);
        x = b.add(POOCH_L_TAIL_PROJ, c3, p, out, out, h2, h2, 0, 1, 0, pre + ".tail", e2);
      } else {
        x = b.add(POOCH_L_TAIL_ID, c3, x, out, out, h2, h2, 0, 1, 0, pre + ".tail", e2);
      }
      e = e2;
      h = h2;
      cin = out;
    }
  }
  int a = b.add(POOCH_L_AVGPOOL, x, -1, cin, cin, 1, 1, 0, 1, 0, "avgpool", 1);
  b.add(POOCH_L_FC_CE, a, -1, cin, classes, 1, 1, 0, 1, 0, "fc", 1);
}

// SURVEY 8(f) f2 (oracle: nets.fuse_bnrelu, same rule): merge every BN-ReLU whose only consumer
// is a single-input 2D conv with cin % 32 == 0 and stride <= 2 into that conv.
void fuse_bnrelu(std::vector<pooch_layer_desc>& L) {
  const int n = (int)L.size();
  std::vector<int> ncons(n, 0), cons(n, -1);
  for (int i = 0; i < n; ++i)
    for (int m : {L[i].in0, L[i].in1})
      if (m >= 0) {
        ncons[m]++;
        cons[m] = i;
      }
  std::vector<char> gone(n, 0);
  for (int i = 0; i < n; ++i) {
    if (L[i].kind != POOCH_L_BNRELU || ncons[i] != 1 || L[i].dout > 0) continue;
    const pooch_layer_desc& u = L[cons[i]];
    if (u.kind == POOCH_L_CONV && u.in0 == i && u.in1 < 0 && u.cin % 32 == 0 && u.stride <= 2) gone[i] = 1;
  }
  std::vector<int> nid(n, -1);
  std::vector<pooch_layer_desc> out;
  for (int i = 0; i < n; ++i) {
    if (gone[i]) continue;
    pooch_layer_desc d = L[i];
    if (d.kind == POOCH_L_CONV && d.in0 >= 0 && gone[d.in0]) {
      const pooch_layer_desc& bn = L[d.in0];
      std::string nm = std::string(bn.name, strnlen(bn.name, sizeof(bn.name))) + "+" +
                       std::string(d.name, strnlen(d.name, sizeof(d.name)));
      std::snprintf(d.name, sizeof(d.name), "%s", nm.c_str());
      d.kind = POOCH_L_BNRELU_CONV;
      d.in0 = L[d.in0].in0;
    }
    if (d.in0 >= 0) d.in0 = nid[d.in0];
    if (d.in1 >= 0) d.in1 = nid[d.in1];
    nid[i] = (int)out.size();
    out.push_back(d);
  }
  L.swap(out);
}

}  // namespace

bool build_graph(const pooch_layer_desc* layers, int n, const pooch_io_desc& io, Graph& g, std::string& err) {
  g.t.clear();
  g.io = io;
  if (n <= 0 || io.batch <= 0 || io.in_c % 4 != 0 || io.in_d < 0) {
    err = "empty graph, bad batch or input channels not a multiple of 4";
    return false;
  }
  const bool three = io.in_d > 0;
  if (three && io.batch != 1) {
    err = "3D networks run at batch 1 (BASELINE config 4)";
    return false;
  }
  for (int i = 0; i < n; ++i) {
    const pooch_layer_desc& d = layers[i];
    Task t{};
    t.kind = d.kind; t.in0 = d.in0; t.in1 = d.in1; t.cin = d.cin; t.cout = d.cout; t.hout = d.hout;
    t.wout = d.wout; t.k = d.k; t.stride = d.stride; t.pad = d.pad;
    t.dout = three ? d.dout : 0;
    t.groups = d.groups > 1 ? d.groups : 1;
    t.stride_d = three ? d.stride_d : 0;
    if ((t.groups > 1 && (d.kind != POOCH_L_CONV || !three || d.cin != d.cout || d.cin % t.groups)) ||
        (t.stride_d > 0 && d.kind != POOCH_L_CONV)) {
      err = "task " + std::to_string(i) + ": groups / depth stride are for 3D convs (grouped: cin == cout)";
      return false;
    }
    t.name = std::string(d.name, strnlen(d.name, sizeof(d.name)));
    if (d.in0 >= i || d.in1 >= i || d.in0 < -1 || d.in1 < -1) {
      err = "task " + std::to_string(i) + ": inputs must be topological";
      return false;
    }
    if (d.kind < POOCH_L_CONV || d.kind > POOCH_L_FC_RELU_DROP) {
      err = "task " + std::to_string(i) + ": bad kind";
      return false;
    }
    if (d.in0 >= 0) t.inputs.push_back(d.in0);
    if (d.in1 >= 0) t.inputs.push_back(d.in1);
    const bool two = d.kind == POOCH_L_TAIL_PROJ || d.kind == POOCH_L_TAIL_ID || (d.kind == POOCH_L_CONV && d.in1 >= 0);
    const bool may_read_input = (d.kind == POOCH_L_CONV && !two) || d.kind == POOCH_L_CONV_RELU;
    if (two != (d.in1 >= 0) || (!may_read_input && d.in0 < 0)) {
      err = "task " + std::to_string(i) + ": wrong number of inputs";
      return false;
    }
    // input spatial dims
    if (d.in0 >= 0) {
      t.hin = g.t[d.in0].hout;
      t.win = g.t[d.in0].wout;
      t.din = g.t[d.in0].dout;
      int cprev = g.t[d.in0].cout;
      if (d.kind == POOCH_L_FC_CE || d.kind == POOCH_L_FC_RELU_DROP) cprev *= t.hin * t.win;
      if (d.kind == POOCH_L_CONV && d.in1 >= 0) {  // two-source conv: same grid, channels concatenated
        const Task& o = g.t[d.in1];
        if (o.hout != t.hin || o.wout != t.win || o.dout != t.din || cprev % 32 || o.cout % 32) {
          err = "task " + std::to_string(i) + ": two-source conv needs equal grids and 32-aligned channels";
          return false;
        }
        cprev += o.cout;
      }
      if (cprev != d.cin) {
        err = "task " + std::to_string(i) + ": cin does not match producer";
        return false;
      }
    } else {
      t.hin = io.in_h;
      t.win = io.in_w;
      t.din = three ? io.in_d : 0;
      if (d.cin != io.in_c) {
        err = "task " + std::to_string(i) + ": cin does not match network input";
        return false;
      }
    }
    if (d.cout % 4 != 0 || d.cin % 4 != 0 || d.cout <= 0 || d.hout <= 0 || d.wout <= 0) {
      if (!((d.kind == POOCH_L_FC_CE || d.kind == POOCH_L_HEAD_CE) && d.cin % 4 == 0 && d.cout > 0)) {
        err = "task " + std::to_string(i) + ": channels must be positive multiples of 4";
        return false;
      }
    }
    if (d.kind == POOCH_L_BNRELU_CONV) {
      const Task& c = g.t[d.in0];
      if (three || c.kind != POOCH_L_CONV && c.kind != POOCH_L_BNRELU_CONV || d.cin % 32 || d.stride > 2) {
        err = "task " + std::to_string(i) + ": BNRELU_CONV needs a 2D conv producer, cin % 32 == 0, stride <= 2";
        return false;
      }
    }
    if ((d.kind == POOCH_L_CONV_RELU || d.kind == POOCH_L_LRN || d.kind == POOCH_L_FC_RELU_DROP) && three) {
      err = "task " + std::to_string(i) + ": the AlexNet kinds are 2D";
      return false;
    }
    if (d.kind == POOCH_L_LRN && (d.cout != d.cin || d.hout != t.hin || d.wout != t.win || d.cin > 1024)) {
      err = "task " + std::to_string(i) + ": LRN keeps the shape (C <= 1024)";
      return false;
    }
    if (d.kind == POOCH_L_FC_RELU_DROP && (d.hout != 1 || d.wout != 1 || d.k < 0 || d.k >= 100)) {
      err = "task " + std::to_string(i) + ": FC_RELU_DROP outputs [batch][cout]; k = drop percent in [0, 100)";
      return false;
    }
    if (d.kind == POOCH_L_CONV || d.kind == POOCH_L_MAXPOOL || d.kind == POOCH_L_BNRELU_CONV ||
        d.kind == POOCH_L_CONV_RELU) {
      const int sd = t.stride_d > 0 ? t.stride_d : d.stride;
      if (co(t.hin, d.k, d.stride, d.pad) != d.hout || co(t.win, d.k, d.stride, d.pad) != d.wout ||
          (three && co(t.din, d.k, sd, d.pad) != t.dout)) {
        err = "task " + std::to_string(i) + ": output shape does not match geometry";
        return false;
      }
    }
    if (three && d.kind == POOCH_L_MAXPOOL &&
        !((d.k == 2 && d.stride == 2 && d.pad == 0) || (d.k == 3 && d.stride == 2 && d.pad == 1))) {
      err = "task " + std::to_string(i) + ": 3D max-pool is k2 s2 p0 (U-Net) or k3 s2 p1 (ResNeXt)";
      return false;
    }
    if (d.kind == POOCH_L_UPCONV && (!three || d.k != 2 || d.stride != 2 || d.hout != 2 * t.hin ||
                                     d.wout != 2 * t.win || t.dout != 2 * t.din)) {
      err = "task " + std::to_string(i) + ": UPCONV is a 3D k2 s2 transposed conv doubling each extent";
      return false;
    }
    if (d.kind == POOCH_L_HEAD_CE && (d.hout != t.hin || d.wout != t.win || t.dout != t.din)) {
      err = "task " + std::to_string(i) + ": the head keeps the grid";
      return false;
    }
    if ((d.kind == POOCH_L_AVGPOOL || d.kind == POOCH_L_FC_CE) && three && (d.dout != 1 || d.hout != 1 || d.wout != 1)) {
      err = "task " + std::to_string(i) + ": a 3D global average pool / FC outputs one voxel (dout = hout = wout = 1)";
      return false;
    }
    if ((d.kind == POOCH_L_FC_CE || d.kind == POOCH_L_HEAD_CE) && i != n - 1) {
      err = "the FC / head + cross-entropy task must be the sink";
      return false;
    }
    // bwd reads (see pooch_layer_kind)
    switch (d.kind) {
      case POOCH_L_CONV:
      case POOCH_L_BNRELU_CONV:
      case POOCH_L_BNRELU:
      case POOCH_L_TAIL_PROJ:
      case POOCH_L_TAIL_ID:
      case POOCH_L_UPCONV:
      case POOCH_L_MAXPOOL:
      case POOCH_L_LRN: t.needs = t.inputs; break;
      case POOCH_L_AVGPOOL: break;
      case POOCH_L_CONV_RELU:
      case POOCH_L_FC_RELU_DROP:   // the ReLU mask comes from the task's own output
        t.needs = t.inputs;
        t.needs.push_back(i);
        break;
      case POOCH_L_FC_CE:
      case POOCH_L_HEAD_CE:
        t.needs = t.inputs;
        t.needs.push_back(i);
        break;
    }
    std::sort(t.needs.begin(), t.needs.end());
    t.map_bytes = (uint64_t)io.batch * d.cout * d.hout * d.wout * (three ? (uint64_t)t.dout : 1ull) * 4ull;
    g.t.push_back(t);
  }
  if (g.t.back().kind != POOCH_L_FC_CE && g.t.back().kind != POOCH_L_HEAD_CE) {
    err = "the last task must be FC / head + cross-entropy";
    return false;
  }
  for (int i = 0; i < n; ++i)
    for (int m : g.t[i].inputs) g.t[m].consumers.push_back(i);
  for (int i = 0; i + 1 < n; ++i)
    if (g.t[i].consumers.empty()) {
      err = "task " + std::to_string(i) + " has no consumer (single-sink DAG required)";
      return false;
    }
  return true;
}

bool problem_from_c(const pooch_problem& p, Problem& o, std::string& err) {
  if (p.n <= 0 || !p.fwd_ns || !p.bwd_ns || !p.d2h_ns || !p.h2d_ns || !p.bytes || !p.in_ptr || !p.in_idx ||
      !p.need_ptr || !p.need_idx) {
    err = "incomplete problem";
    return false;
  }
  o.n = p.n;
  o.fwd.assign(p.fwd_ns, p.fwd_ns + p.n);
  o.bwd.assign(p.bwd_ns, p.bwd_ns + p.n);
  o.rec.assign(p.rec_ns ? p.rec_ns : p.fwd_ns, (p.rec_ns ? p.rec_ns : p.fwd_ns) + p.n);
  o.d2h.assign(p.d2h_ns, p.d2h_ns + p.n);
  o.h2d.assign(p.h2d_ns, p.h2d_ns + p.n);
  o.bytes.assign(p.bytes, p.bytes + p.n);
  o.inputs.assign(p.n, {});
  o.needs.assign(p.n, {});
  for (int i = 0; i < p.n; ++i) {
    if (o.fwd[i] <= 0 || o.bwd[i] <= 0 || o.rec[i] <= 0 || o.d2h[i] <= 0 || o.h2d[i] <= 0) {
      err = "durations must be positive (task " + std::to_string(i) + ")";
      return false;
    }
    for (int k = p.in_ptr[i]; k < p.in_ptr[i + 1]; ++k) {
      int m = p.in_idx[k];
      if (m < 0) continue;
      if (m >= i) {
        err = "task " + std::to_string(i) + ": inputs must be topological";
        return false;
      }
      o.inputs[i].push_back(m);
    }
    for (int k = p.need_ptr[i]; k < p.need_ptr[i + 1]; ++k) {
      int m = p.need_idx[k];
      if (m < 0 || m > i) {
        err = "task " + std::to_string(i) + ": needs out of range";
        return false;
      }
      o.needs[i].push_back(m);
    }
    std::sort(o.needs[i].begin(), o.needs[i].end());
    o.needs[i].erase(std::unique(o.needs[i].begin(), o.needs[i].end()), o.needs[i].end());
  }
  o.resident = p.resident_bytes;
  o.budget = p.budget_bytes;
  o.tail = p.tail_ns;
  o.host_budget = p.host_budget_bytes;
  if (p.duplex_d2h_permille < 0 || p.duplex_d2h_permille > 1000 || p.duplex_h2d_permille < 0 ||
      p.duplex_h2d_permille > 1000) {
    err = "duplex_*_permille must be in 0..1000";
    return false;
  }
  o.duplex_d2h = p.duplex_d2h_permille > 0 ? p.duplex_d2h_permille : 1000;
  o.duplex_h2d = p.duplex_h2d_permille > 0 ? p.duplex_h2d_permille : 1000;
  o.is_conv.assign(p.n, 0);
  if (p.is_conv)
    for (int i = 0; i < p.n; ++i) o.is_conv[i] = p.is_conv[i] ? 1 : 0;
  return true;
}

}  // namespace pooch

using namespace pooch;

extern "C" pooch_status pooch_build_net(int32_t which, int32_t in_hw, int32_t classes, int32_t width,
                                        pooch_layer_desc* out, int32_t* n_layers) {
  if (!n_layers) return fail(POOCH_EUSAGE, "n_layers is null");
  const bool fuse = (which & POOCH_NET_FUSE_BNRELU) != 0;
  which &= ~POOCH_NET_FUSE_BNRELU;
  Builder b;
  if (which == 0) {
    if (in_hw <= 0 || in_hw % 2 || width <= 0 || width % 4) return fail(POOCH_EUSAGE, "bad tiny CNN size");
    tiny(b, in_hw, classes, width);
  } else if (which == 1 || which == 2) {
    if (in_hw < 32) return fail(POOCH_EUSAGE, "ResNet-50 input too small");
    resnet50(b, in_hw, classes, which == 1);
  } else if (which == 3) {
    if (in_hw < 16 || in_hw % 16 || width <= 0 || width % 32) return fail(POOCH_EUSAGE, "bad 3D U-Net size");
    unet3d(b, in_hw, classes, width);
  } else if (which == 4) {
    if (in_hw < 67) return fail(POOCH_EUSAGE, "AlexNet input too small (>= 67)");
    alexnet(b, in_hw, classes);
  } else if (which == 5 || which == 6) {
    if (in_hw < 32 || width < 8) return fail(POOCH_EUSAGE, "ResNeXt (3D) input too small (H = W >= 32, D >= 8)");
    resnext3d(b, width, in_hw, classes, which == 5 ? 101 : 50);
  } else {
    return fail(POOCH_EUSAGE, "unknown network %d", which);
  }
  if (fuse) fuse_bnrelu(b.out);
  int n = (int)b.out.size();
  if (out) {
    if (*n_layers < n) return fail(POOCH_EUSAGE, "output array too small (%d < %d)", *n_layers, n);
    std::copy(b.out.begin(), b.out.end(), out);
  }
  *n_layers = n;
  return POOCH_OK;
}
