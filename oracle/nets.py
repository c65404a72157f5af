"""The two CNN workloads as fused task lists, their fp64 training step, and the
saved-feature-map census (oracle, C1 + C2).

A *task* is one executor kernel group; a *feature map* is a task's output that
backward needs (Sec. 2.1: "Computation of backward-propagation of layer
i requires the feature maps, which has been computed in forward propagation of
layer i"). PoocH classifies feature maps only (Sec. 4.1.1). Reading 1:
maps = conv outputs, BN(+add)+ReLU outputs, pool outputs and the FC output;
for ResNet-50 this census gives 105, the row total of every Table 3 line
(P:L443-446).

Task kinds (inputs are map ids, -1 = the network input, which is not a map
and is always resident, Reading 2):

* ``conv``      y = conv(x, W)                 bwd needs {x}
* ``bnrelu``    y = relu(bn(c))                bwd needs {c} (mask from bn(c))
* ``tail_proj`` y = relu(bn3(c3) + bnp(p))     bwd needs {c3, p}
* ``tail_id``   y = relu(bn3(c3) + x)          bwd needs {c3, x}
* ``maxpool``   y = maxpool(x)                 bwd needs {x} (argmax from x)
* ``avgpool``   y = mean_hw(x)                 bwd needs {}
* ``fc_ce``     z = flat(x) W^T + b; CE loss   bwd needs {x, z} (sink task)
* ``bnrelu_conv``  y = conv(relu(bn(c)), W)    bwd needs {c}  (the BN-ReLU
  applied to the conv's operand on load, so relu(bn(c)) is never a map; built by
  ``fuse_bnrelu`` from the plain graph, same function, same parameters)

3D network (BASELINE.json config 4, "3D U-Net-style, conv3d-BN-ReLU"):

* ``conv`` with two inputs    y = conv3d(concat_c(a, b), W)  bwd needs {a, b}
* ``upconv``    y = transposed conv3d k2 s2 (up-sampling)     bwd needs {x}
* ``maxpool``   (3D) k2 s2 over 2x2x2 windows               bwd needs {x}
* ``head_ce``   z = x W^T + b per voxel; CE averaged over voxels   bwd needs {x, z} (sink)

Flatten order before the FC is (h, w, c) (the GPU's NHWC order); both sides
use it, so FC weights are shared verbatim.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import layers as L

import synthdata


@dataclass
class Task:
    name: str
    kind: str
    inputs: list            # map ids (task ids), -1 = network input
    out_chw: tuple          # per-image output shape (C, H, W) -- (C, D, H, W) in 3D nets; FC/avgpool: (C, 1, 1)
    stride: int = 1
    pad: int = 0
    k: int = 0              # conv/pool kernel size
    cin: int = 0            # conv input channels (true, unpadded)
    bn: str = ""            # bnrelu_conv: name of the fused BN-ReLU (its gamma / beta)
    ratio: float = 0.0      # fc_relu_drop: dropout probability
    groups: int = 1         # conv: grouped convolution (ResNeXt's cardinality), w is [O, cin/groups, k..]
    stride_d: int = 0       # 3D conv: stride along depth (0: = stride); ResNeXt-101 (3D)'s stem is (1, 2, 2)

    @property
    def stride3(self):
        return (self.stride_d or self.stride, self.stride, self.stride)

    @property
    def needs(self):
        """Maps bwd(task) reads (see module docstring)."""
        if self.kind in ("conv", "maxpool", "upconv", "bnrelu_conv", "lrn"):
            return [i for i in self.inputs if i >= 0]
        if self.kind in ("conv_relu", "fc_relu_drop"):
            return None     # filled by Net (self id needed: the ReLU mask comes from the output)
        if self.kind in ("bnrelu", "tail_proj", "tail_id"):
            return [i for i in self.inputs if i >= 0]
        if self.kind == "avgpool":
            return []
        if self.kind in ("fc_ce", "head_ce"):
            return None     # filled by Net (self id needed)
        raise ValueError(self.kind)


@dataclass
class Net:
    name: str
    in_chw: tuple           # (C, H, W) of the network input, unpadded; (C, D, H, W) in 3D
    classes: int
    tasks: list = field(default_factory=list)

    @property
    def dims(self):
        return len(self.in_chw) - 1

    def add(self, t: Task) -> int:
        self.tasks.append(t)
        return len(self.tasks) - 1

    def needs(self, i):
        t = self.tasks[i]
        if t.kind in ("fc_ce", "head_ce", "conv_relu", "fc_relu_drop"):
            return sorted([j for j in t.inputs if j >= 0] + [i])
        return sorted(t.needs)

    def map_bytes_per_image(self, i):
        return 4 * int(np.prod(self.tasks[i].out_chw))


# ------------------------------------------------------------------ builders
def tiny_cnn(width: int = 32, in_hw: int = 32, classes: int = 10) -> Net:
    """BASELINE.json config 1: 4 x [conv3x3-BN-ReLU] (uniform width 32, SURVEY
    8(d)), maxpool 2x2, FC-10."""
    net = Net("tiny", (3, in_hw, in_hw), classes)
    src, cin, hw = -1, 3, in_hw
    for l in range(4):
        c = net.add(Task(f"conv{l}", "conv", [src], (width, hw, hw), 1, 1, 3, cin))
        src = net.add(Task(f"bn{l}", "bnrelu", [c], (width, hw, hw)))
        cin = width
    hw2 = hw // 2
    p = net.add(Task("maxpool", "maxpool", [src], (width, hw2, hw2), 2, 0, 2))
    net.add(Task("fc", "fc_ce", [p], (classes, 1, 1), cin=width * hw2 * hw2))
    return net


def resnet50(in_hw: int = 224, classes: int = 1000, v15: bool = True) -> Net:
    """ResNet-50 [resnet]; v1.5 (stride on the 3x3) by default
    (Reading 24)."""
    net = Net("resnet50" if v15 else "resnet50v1", (3, in_hw, in_hw), classes)
    hw = L.conv_out_hw(in_hw, in_hw, 7, 7, 2, 3)[0]
    c = net.add(Task("conv1", "conv", [-1], (64, hw, hw), 2, 3, 7, 3))
    x = net.add(Task("bn1", "bnrelu", [c], (64, hw, hw)))
    hw = L.conv_out_hw(hw, hw, 3, 3, 2, 1)[0]
    x = net.add(Task("maxpool", "maxpool", [x], (64, hw, hw), 2, 1, 3))
    cin = 64
    for si, (nblocks, mid) in enumerate(zip([3, 4, 6, 3], [64, 128, 256, 512])):
        out = 4 * mid
        for b in range(nblocks):
            s = 2 if (b == 0 and si > 0) else 1
            pre = f"layer{si + 1}.{b}"
            s1, s2 = (1, s) if v15 else (s, 1)
            hw1 = L.conv_out_hw(hw, hw, 1, 1, s1, 0)[0]
            c1 = net.add(Task(pre + ".conv1", "conv", [x], (mid, hw1, hw1), s1, 0, 1, cin))
            y1 = net.add(Task(pre + ".bn1", "bnrelu", [c1], (mid, hw1, hw1)))
            hw2 = L.conv_out_hw(hw1, hw1, 3, 3, s2, 1)[0]
            c2 = net.add(Task(pre + ".conv2", "conv", [y1], (mid, hw2, hw2), s2, 1, 3, mid))
            y2 = net.add(Task(pre + ".bn2", "bnrelu", [c2], (mid, hw2, hw2)))
            c3 = net.add(Task(pre + ".conv3", "conv", [y2], (out, hw2, hw2), 1, 0, 1, mid))
            if b == 0:
                p = net.add(Task(pre + ".downsample", "conv", [x], (out, hw2, hw2), s, 0, 1, cin))
                x = net.add(Task(pre + ".tail", "tail_proj", [c3, p], (out, hw2, hw2)))
            else:
                x = net.add(Task(pre + ".tail", "tail_id", [c3, x], (out, hw2, hw2)))
            hw, cin = hw2, out
    a = net.add(Task("avgpool", "avgpool", [x], (cin, 1, 1)))
    net.add(Task("fc", "fc_ce", [a], (classes, 1, 1), cin=cin))
    return net


def alexnet(in_hw: int = 227, classes: int = 1000, drop: float = 0.5) -> Net:
    """AlexNet [alexnet], the paper's compute-heavy workload, in the
    single-tower form of Chainer's example: conv1 11x11/4 (96) -> ReLU -> LRN -> max-pool 3/2;
    conv2 5x5 pad 2 (256) -> ReLU -> LRN -> max-pool 3/2; conv3 3x3 (384), conv4 3x3 (384),
    conv5 3x3 (256) each -> ReLU, max-pool 3/2 after conv5; fc6 (4096), fc7 (4096) each -> ReLU ->
    dropout; fc8 (classes) -> softmax CE. Convolutions and FC layers carry biases. Tasks:
    ``conv_relu`` y = relu(conv(x) + b) (bwd needs {x, y}), ``lrn`` (bwd needs {x}), ``maxpool``,
    ``fc_relu_drop`` y = dropout(relu(x W^T + b)) (bwd needs {x, y}), ``fc_ce``. 13 maps."""
    net = Net("alexnet", (3, in_hw, in_hw), classes)

    def co(h, k, s, p):
        return (h + 2 * p - k) // s + 1

    h = co(in_hw, 11, 4, 0)
    x = net.add(Task("conv1", "conv_relu", [-1], (96, h, h), 4, 0, 11, 3))
    x = net.add(Task("lrn1", "lrn", [x], (96, h, h)))
    h = co(h, 3, 2, 0)
    x = net.add(Task("pool1", "maxpool", [x], (96, h, h), 2, 0, 3))
    x = net.add(Task("conv2", "conv_relu", [x], (256, h, h), 1, 2, 5, 96))
    x = net.add(Task("lrn2", "lrn", [x], (256, h, h)))
    h = co(h, 3, 2, 0)
    x = net.add(Task("pool2", "maxpool", [x], (256, h, h), 2, 0, 3))
    x = net.add(Task("conv3", "conv_relu", [x], (384, h, h), 1, 1, 3, 256))
    x = net.add(Task("conv4", "conv_relu", [x], (384, h, h), 1, 1, 3, 384))
    x = net.add(Task("conv5", "conv_relu", [x], (256, h, h), 1, 1, 3, 384))
    h = co(h, 3, 2, 0)
    x = net.add(Task("pool5", "maxpool", [x], (256, h, h), 2, 0, 3))
    x = net.add(Task("fc6", "fc_relu_drop", [x], (4096, 1, 1), cin=256 * h * h, ratio=drop))
    x = net.add(Task("fc7", "fc_relu_drop", [x], (4096, 1, 1), cin=4096, ratio=drop))
    net.add(Task("fc8", "fc_ce", [x], (classes, 1, 1), cin=4096))
    return net


def unet3d(in_d: int = 256, width: int = 256, classes: int = 2, cin: int = 1) -> Net:
    """BASELINE.json config 4 / SURVEY 8(d): a 3D U-Net -- 4 levels of widths w, 2w, 4w,
    4w (256/512/1024/1024 at w = 256), each 2 x [conv3d 3^3 -> BN -> ReLU]; 2^3 max-pool
    between levels; a 4w bottleneck; decoder levels up-sample with a k2 s2 transposed conv
    to the level's width, concatenate the skip (read as a second input of the first conv)
    and apply 2 x [conv3d -> BN -> ReLU]; a 1^3 head to ``classes`` with per-voxel softmax
    cross-entropy. 45 maps; 207.2 GB at 256^3."""
    net = Net("unet3d", (cin, in_d, in_d, in_d), classes)
    widths = [width, 2 * width, 4 * width, 4 * width]
    src, c, e = -1, cin, in_d
    skips = []

    def block(pre, x, cin_, w, e_):
        c1 = net.add(Task(pre + ".conv1", "conv", x, (w, e_, e_, e_), 1, 1, 3, cin_))
        y1 = net.add(Task(pre + ".bn1", "bnrelu", [c1], (w, e_, e_, e_)))
        c2 = net.add(Task(pre + ".conv2", "conv", [y1], (w, e_, e_, e_), 1, 1, 3, w))
        return net.add(Task(pre + ".bn2", "bnrelu", [c2], (w, e_, e_, e_)))

    for lv, w in enumerate(widths):
        y = block(f"enc{lv + 1}", [src], c, w, e)
        skips.append((y, w, e))
        e //= 2
        src = net.add(Task(f"pool{lv + 1}", "maxpool", [y], (w, e, e, e), 2, 0, 2))
        c = w
    src = block("mid", [src], c, widths[-1], e)
    c = widths[-1]
    for lv in reversed(range(4)):
        sk, w, e = skips[lv]
        u = net.add(Task(f"up{lv + 1}", "upconv", [src], (w, e, e, e), 2, 0, 2, c))
        src = block(f"dec{lv + 1}", [u, sk], 2 * w, w, e)
        c = w
    net.add(Task("head", "head_ce", [src], (classes, e, e, e), cin=c))
    return net


def resnext3d(in_dhw=(16, 112, 112), classes: int = 400, depth: int = 101, cardinality: int = 32,
              cin: int = 3, widths=(128, 256, 512, 1024), blocks=None, stem: int = 64) -> Net:
    """ResNeXt-101 (3D), the paper's third workload (Sec. 5.2; SURVEY 8(f)
    f4), as [3dnn] builds it from ResNeXt [resnext]: conv 7^3 (stride (1, 2, 2), pad 3, 64) ->
    BN -> ReLU -> max-pool 3^3 / 2 (pad 1); four stages of [3, 4, 23, 3] bottleneck blocks of
    widths 128 / 256 / 512 / 1024 (= cardinality 32 x 4 / 8 / 16 / 32 channels per group):
    conv 1^3 -> BN -> ReLU -> GROUPED conv 3^3 (32 groups; stride 2 in the first block of stages
    2-4) -> BN -> ReLU -> conv 1^3 to twice the width -> BN, plus the shortcut (a 1^3 projection
    conv + BN in each stage's first block, "shortcut type B"), -> add -> ReLU; global average
    pool; FC to ``classes``. Task kinds are ResNet-50's (the bottleneck's tails, BN-ReLU
    groups, pools); only the 3D geometry and the groups differ. depth 50: [3, 4, 6, 3].
    ``widths`` / ``blocks`` / ``stem`` / ``cardinality`` shrink it for the finite-difference
    pins (tests only)."""
    blocks = blocks or {50: [3, 4, 6, 3], 101: [3, 4, 23, 3]}[depth]
    d, h, w = in_dhw
    net = Net("resnext%d_3d" % depth, (cin,) + tuple(in_dhw), classes)

    def out3(dhw, k, s3, p):
        return L.gconv3d_out(dhw, k, s3, p)
    e = out3((d, h, w), 7, (1, 2, 2), 3)
    c = net.add(Task("conv1", "conv", [-1], (stem,) + e, 2, 3, 7, cin, stride_d=1))
    x = net.add(Task("bn1", "bnrelu", [c], (stem,) + e))
    e = out3(e, 3, 2, 1)
    x = net.add(Task("maxpool", "maxpool", [x], (stem,) + e, 2, 1, 3))
    cin_ = stem
    for si, (nb, mid) in enumerate(zip(blocks, widths)):
        out = 2 * mid
        for b in range(nb):
            s = 2 if (b == 0 and si > 0) else 1
            pre = f"layer{si + 1}.{b}"
            c1 = net.add(Task(pre + ".conv1", "conv", [x], (mid,) + e, 1, 0, 1, cin_))
            y1 = net.add(Task(pre + ".bn1", "bnrelu", [c1], (mid,) + e))
            e2 = out3(e, 3, s, 1)
            c2 = net.add(Task(pre + ".conv2", "conv", [y1], (mid,) + e2, s, 1, 3, mid, groups=cardinality))
            y2 = net.add(Task(pre + ".bn2", "bnrelu", [c2], (mid,) + e2))
            c3 = net.add(Task(pre + ".conv3", "conv", [y2], (out,) + e2, 1, 0, 1, mid))
            if b == 0:
                p = net.add(Task(pre + ".downsample", "conv", [x], (out,) + e2, s, 0, 1, cin_))
                x = net.add(Task(pre + ".tail", "tail_proj", [c3, p], (out,) + e2))
            else:
                x = net.add(Task(pre + ".tail", "tail_id", [c3, x], (out,) + e2))
            e, cin_ = e2, out
    a = net.add(Task("avgpool", "avgpool", [x], (cin_, 1, 1)))
    net.add(Task("fc", "fc_ce", [a], (classes, 1, 1), cin=cin_))
    return net


def fuse_bnrelu(net: Net) -> Net:
    """merge every ``bnrelu`` whose only consumer is a single-input 2D conv with
    32-multiple input channels (the B200 path's TMA-fed operand loader, which applies the
    BN-ReLU on load) into that conv (kind ``bnrelu_conv``). Same function and parameters; the
    merged BN-ReLU outputs stop being maps. Task order is kept; inputs are renumbered."""
    n = len(net.tasks)
    consumers = [[k for k in range(n) if i in net.tasks[k].inputs] for i in range(n)]
    fused = set()
    for i, t in enumerate(net.tasks):
        if t.kind != "bnrelu" or len(consumers[i]) != 1 or net.dims != 2:
            continue
        k = consumers[i][0]
        u = net.tasks[k]
        if u.kind == "conv" and u.inputs == [i] and u.cin % 32 == 0 and u.stride <= 2:
            fused.add(i)
    out = Net(net.name + "_f2", net.in_chw, net.classes)
    new_id = {}
    for i, t in enumerate(net.tasks):
        if i in fused:
            continue
        ins = []
        for j in t.inputs:
            ins.append(-1 if j < 0 else new_id[net.tasks[j].inputs[0] if j in fused else j])
        if t.kind == "conv" and t.inputs[0] in fused:
            bn = net.tasks[t.inputs[0]]
            nt = Task(t.name, "bnrelu_conv", ins, t.out_chw, t.stride, t.pad, t.k, t.cin, bn=bn.name)
        else:
            nt = Task(t.name, t.kind, ins, t.out_chw, t.stride, t.pad, t.k, t.cin, t.bn)
        new_id[i] = out.add(nt)
    return out


# -------------------------------------------------------------------- census
def census(net: Net, batch: int):
    """[(name, bytes)] of every saved feature map (C2)."""
    return [(t.name, batch * net.map_bytes_per_image(i)) for i, t in enumerate(net.tasks)]


def param_shapes(net: Net):
    """Ordered {param name: shape}; conv weights OIHW, FC [O, I]."""
    shapes = {}
    for t in net.tasks:
        if t.kind == "bnrelu_conv":     # the fused BN's parameters first (the plain graph's order)
            shapes[t.bn + ".gamma"] = (t.cin,)
            shapes[t.bn + ".beta"] = (t.cin,)
        if t.kind in ("conv", "bnrelu_conv", "conv_relu"):
            shapes[t.name + ".w"] = (t.out_chw[0], t.cin // t.groups) + (t.k,) * (len(t.out_chw) - 1)
            if t.kind == "conv_relu":
                shapes[t.name + ".b"] = (t.out_chw[0],)
        elif t.kind == "fc_relu_drop":
            shapes[t.name + ".w"] = (t.out_chw[0], t.cin)
            shapes[t.name + ".b"] = (t.out_chw[0],)
        elif t.kind == "upconv":
            shapes[t.name + ".w"] = (t.cin, t.out_chw[0], 2, 2, 2)
        elif t.kind == "bnrelu":
            shapes[t.name + ".gamma"] = (t.out_chw[0],)
            shapes[t.name + ".beta"] = (t.out_chw[0],)
        elif t.kind in ("tail_proj", "tail_id"):
            shapes[t.name + ".gamma3"] = (t.out_chw[0],)
            shapes[t.name + ".beta3"] = (t.out_chw[0],)
            if t.kind == "tail_proj":
                shapes[t.name + ".gammap"] = (t.out_chw[0],)
                shapes[t.name + ".betap"] = (t.out_chw[0],)
        elif t.kind in ("fc_ce", "head_ce"):
            shapes[t.name + ".w"] = (t.out_chw[0], t.cin)
            shapes[t.name + ".b"] = (t.out_chw[0],)
    return shapes


# ------------------------------------------------------------ training step
def _flat_hwc(x):
    return x.transpose(0, 2, 3, 1).reshape(x.shape[0], -1)


def forward_backward(net: Net, params: dict, x_nhwc: np.ndarray, labels: np.ndarray, map_grads=None,
                     precision: str = "fp64", rng=(0, 0), decisions=None):
    """One fp64 fwd + bwd of ``net``. ``x_nhwc`` is the (unpadded)
    input batch in NHWC; params are promoted to fp64. Returns (loss, grads,
    outputs) with grads keyed like ``params`` and outputs the fp64 task
    outputs (NCHW) for map-level checks; ``map_grads`` (a list) receives the
    gradient of every map. ``precision="tf32"`` rounds the operands of every
    contraction (conv fwd / dgrad / wgrad, FC) with ``layers.tf32`` -- the
    kernels' operand precision -- and keeps everything else in fp64.
    ``rng`` = (seed, step) of the counter-based dropout masks (``layers.dropout_keep``, salted
    with the task id). ``precision="fp32"`` runs the same code with every array in fp32 (NumPy
    keeps fp32 through every layer call; the contractions are fp32 BLAS): the
    oracle's fp32 mode, which measures how far plain fp32 arithmetic alone
    moves a result from fp64 (DESIGN.md Reading 28).
    ``decisions`` ({task id: NCHW array}, optional) takes the discrete choices from given tensors
    -- the GPU's own forward maps -- instead of this run's values: for ReLU-type tasks (bnrelu,
    tail_*, conv_relu, fc_relu_drop) the ReLU mask is [given output > 0]; for max-pool tasks the
    window winners are the first maxima of the given INPUT map. Everything else stays fp64, so
    both sides decide in the same precision (layers.maxpool_argmax)."""
    q = L.tf32 if precision == "tf32" else (lambda a: a)
    dt = np.float32 if precision == "fp32" else np.float64
    P = {k: np.asarray(v, dtype=dt) for k, v in params.items()}
    x_np = np.asarray(x_nhwc, dtype=dt)
    x_in = np.moveaxis(x_np, -1, 1)          # N(D)HWC -> NC(D)HW
    three = net.dims == 3
    outs, caches = [], []
    dec = decisions or {}
    masks = {}           # task id -> ReLU mask taken from ``decisions``

    def get(i):
        return x_in if i < 0 else outs[i]

    def conv_in(t):   # a conv with two inputs reads their channel concatenation
        return np.concatenate([get(i) for i in t.inputs], axis=1) if len(t.inputs) > 1 else get(t.inputs[0])

    def _relu_dec(z, i):   # relu(z), or z masked by the given map's positives (decisions)
        if i not in dec:
            return L.relu_fwd(z)
        masks[i] = np.asarray(dec[i]).reshape(z.shape) > 0
        return z * masks[i]

    def _relu_bwd_dec(dy, i):
        return dy * masks[i] if i in masks else L.relu_bwd(dy, outs[i])

    loss = None
    for t in net.tasks:
        if t.kind == "conv" and three and (t.groups > 1 or t.stride_d):
            y = L.gconv3d_fwd(q(conv_in(t)), q(P[t.name + ".w"]), t.stride3, t.pad, t.groups)
            cache = None
        elif t.kind == "conv":
            f = L.conv3d_fwd if three else L.conv2d_fwd
            y = f(q(conv_in(t)), q(P[t.name + ".w"]), t.stride, t.pad)
            cache = None
        elif t.kind == "bnrelu_conv":
            z, bc = L.bn_fwd(get(t.inputs[0]), P[t.bn + ".gamma"], P[t.bn + ".beta"])
            r = L.relu_fwd(z)
            y = L.conv2d_fwd(q(r), q(P[t.name + ".w"]), t.stride, t.pad)
            cache = (bc, r)
        elif t.kind == "upconv":
            y = L.upconv3d_fwd(q(get(t.inputs[0])), q(P[t.name + ".w"]))
            cache = None
        elif t.kind == "head_ce":
            xin = get(t.inputs[0])
            xf = np.moveaxis(xin, 1, -1).reshape(-1, xin.shape[1])         # [voxels, C]
            z = L.fc_fwd(q(xf), q(P[t.name + ".w"]), P[t.name + ".b"])
            loss, dz = L.softmax_ce(z, np.asarray(labels).reshape(-1))
            y = np.moveaxis(z.reshape(xin.shape[:1] + xin.shape[2:] + (z.shape[1],)), -1, 1)
            cache = (xf, dz)
        elif t.kind == "bnrelu":
            z, bc = L.bn_fwd(get(t.inputs[0]), P[t.name + ".gamma"], P[t.name + ".beta"])
            y = _relu_dec(z, len(outs))
            cache = (bc,)
        elif t.kind in ("tail_proj", "tail_id"):
            z3, bc3 = L.bn_fwd(get(t.inputs[0]), P[t.name + ".gamma3"], P[t.name + ".beta3"])
            if t.kind == "tail_proj":
                zp, bcp = L.bn_fwd(get(t.inputs[1]), P[t.name + ".gammap"], P[t.name + ".betap"])
            else:
                zp, bcp = get(t.inputs[1]), None
            y = _relu_dec(z3 + zp, len(outs))
            cache = (bc3, bcp)
        elif t.kind == "maxpool" and len(outs) in dec:
            xd = np.asarray(dec[len(outs)], np.float64)
            arg = (L.maxpool3d_argmax(xd, t.k, t.stride, t.pad) if three
                   else L.maxpool_argmax(xd, t.k, t.stride, t.pad))
            y = (L.maxpool3d_fwd_at(get(t.inputs[0]), arg, t.k, t.stride, t.pad) if three
                 else L.maxpool_fwd_at(get(t.inputs[0]), arg, t.k, t.stride, t.pad))
            cache = arg
        elif t.kind == "maxpool":
            y = (L.maxpool3d_fwd(get(t.inputs[0]), t.k, t.stride, t.pad) if three
                 else L.maxpool_fwd(get(t.inputs[0]), t.k, t.stride, t.pad))
            cache = None
        elif t.kind == "conv_relu":
            y = _relu_dec(L.conv2d_bias_fwd(q(get(t.inputs[0])), q(P[t.name + ".w"]), P[t.name + ".b"],
                                            t.stride, t.pad), len(outs))
            cache = None
        elif t.kind == "lrn":
            y, _ = L.lrn_fwd(get(t.inputs[0]))
            cache = None
        elif t.kind == "fc_relu_drop":
            xf = _flat_hwc(get(t.inputs[0]))
            keep = L.dropout_keep((xf.shape[0], t.out_chw[0]), t.ratio, rng[0], rng[1], len(outs))
            if len(outs) in dec:     # the GPU's kept-and-positive units decide (keep & [z > 0])
                keep = np.asarray(dec[len(outs)]).reshape(xf.shape[0], -1) > 0
                z = L.fc_fwd(q(xf), q(P[t.name + ".w"]), P[t.name + ".b"])
                yf = np.where(keep, z / (1.0 - t.ratio), 0.0)
                z = np.where(keep, np.abs(z) + 1.0, -1.0)   # the mask fc_relu_dropout_bwd applies
            else:
                yf, z = L.fc_relu_dropout_fwd(q(xf), q(P[t.name + ".w"]), P[t.name + ".b"], keep, t.ratio)
            y = yf[:, :, None, None]
            cache = (xf, z, keep)
        elif t.kind == "avgpool":
            y = L.avgpool_fwd(get(t.inputs[0]))[:, :, None, None]     # 3D nets too: [n, c, 1, 1]
            cache = None
        elif t.kind == "fc_ce":
            xf = _flat_hwc(get(t.inputs[0]))
            z = L.fc_fwd(q(xf), q(P[t.name + ".w"]), P[t.name + ".b"])
            loss, dz = L.softmax_ce(z, np.asarray(labels))
            y = z[:, :, None, None]
            cache = (xf, dz)
        else:
            raise ValueError(t.kind)
        outs.append(y)
        caches.append(cache)

    grads = {k: np.zeros_like(v) for k, v in P.items()}
    gmap = [None] * len(net.tasks)

    def acc(i, g):
        if i < 0:
            return
        gmap[i] = g if gmap[i] is None else gmap[i] + g

    for i in reversed(range(len(net.tasks))):
        t = net.tasks[i]
        cache = caches[i]
        if t.kind == "fc_ce":
            xf, dz = cache
            dxf, dw, db = L.fc_bwd(q(dz), q(xf), q(P[t.name + ".w"]))
            db = dz.sum(axis=0)
            grads[t.name + ".w"] += dw
            grads[t.name + ".b"] += db
            src = get(t.inputs[0])
            n, c, h, w = src.shape
            acc(t.inputs[0], dxf.reshape(n, h, w, c).transpose(0, 3, 1, 2))
            continue
        if t.kind == "head_ce":
            xf, dz = cache
            dxf, dw, _ = L.fc_bwd(q(dz), q(xf), q(P[t.name + ".w"]))
            grads[t.name + ".w"] += dw
            grads[t.name + ".b"] += dz.sum(axis=0)
            src = get(t.inputs[0])
            acc(t.inputs[0], np.moveaxis(dxf.reshape(src.shape[:1] + src.shape[2:] + (src.shape[1],)), -1, 1))
            continue
        dy = gmap[i]
        if t.kind == "conv":
            xin = conv_in(t)
            w = P[t.name + ".w"]
            if three and (t.groups > 1 or t.stride_d):
                g_, s_ = t.groups, t.stride3
                fw = lambda a, b, sh, st, pd: L.gconv3d_wgrad(a, b, sh, s_, pd, g_)  # noqa: E731
                fd = lambda a, b, sh, st, pd: L.gconv3d_dgrad(a, b, sh, s_, pd, g_)  # noqa: E731
            else:
                fw, fd = (L.conv3d_wgrad, L.conv3d_dgrad) if three else (L.conv2d_wgrad, L.conv2d_dgrad)
            grads[t.name + ".w"] += fw(q(xin), q(dy), w.shape, t.stride, t.pad)
            if t.inputs[0] >= 0:
                dx = fd(q(dy), q(w), xin.shape, t.stride, t.pad)
                c0 = 0
                for j in t.inputs:          # split the concatenation's gradient per input
                    cj = get(j).shape[1]
                    acc(j, dx[:, c0:c0 + cj])
                    c0 += cj
        elif t.kind == "bnrelu_conv":
            bc, r = cache
            w = P[t.name + ".w"]
            grads[t.name + ".w"] += L.conv2d_wgrad(q(r), q(dy), w.shape, t.stride, t.pad)
            dr = L.conv2d_dgrad(q(dy), q(w), r.shape, t.stride, t.pad)
            dz = L.relu_bwd(dr, r)
            dx, dg, db = L.bn_bwd(dz, bc, P[t.bn + ".gamma"])
            grads[t.bn + ".gamma"] += dg
            grads[t.bn + ".beta"] += db
            acc(t.inputs[0], dx)
        elif t.kind == "upconv":
            dx, dw = L.upconv3d_bwd(q(dy), q(get(t.inputs[0])), q(P[t.name + ".w"]))
            grads[t.name + ".w"] += dw
            acc(t.inputs[0], dx)
        elif t.kind == "bnrelu":
            dz = _relu_bwd_dec(dy, i)
            dx, dg, db = L.bn_bwd(dz, cache[0], P[t.name + ".gamma"])
            grads[t.name + ".gamma"] += dg
            grads[t.name + ".beta"] += db
            acc(t.inputs[0], dx)
        elif t.kind in ("tail_proj", "tail_id"):
            dz = _relu_bwd_dec(dy, i)
            dx3, dg3, db3 = L.bn_bwd(dz, cache[0], P[t.name + ".gamma3"])
            grads[t.name + ".gamma3"] += dg3
            grads[t.name + ".beta3"] += db3
            acc(t.inputs[0], dx3)
            if t.kind == "tail_proj":
                dxp, dgp, dbp = L.bn_bwd(dz, cache[1], P[t.name + ".gammap"])
                grads[t.name + ".gammap"] += dgp
                grads[t.name + ".betap"] += dbp
                acc(t.inputs[1], dxp)
            else:
                acc(t.inputs[1], dz)
        elif t.kind == "maxpool" and cache is not None:      # winners from ``decisions``
            shape = get(t.inputs[0]).shape
            acc(t.inputs[0], L.maxpool3d_bwd_at(dy, shape, cache, t.k, t.stride, t.pad) if three
                else L.maxpool_bwd_at(dy, shape, cache, t.k, t.stride, t.pad))
        elif t.kind == "maxpool":
            acc(t.inputs[0], L.maxpool3d_bwd(dy, get(t.inputs[0]), t.k, t.stride, t.pad) if three
                else L.maxpool_bwd(dy, get(t.inputs[0]), t.k, t.stride, t.pad))
        elif t.kind == "conv_relu":
            dz = _relu_bwd_dec(dy, i)
            xin = get(t.inputs[0])
            w = P[t.name + ".w"]
            grads[t.name + ".w"] += L.conv2d_wgrad(q(xin), q(dz), w.shape, t.stride, t.pad)
            grads[t.name + ".b"] += dz.sum(axis=(0, 2, 3))
            if t.inputs[0] >= 0:
                acc(t.inputs[0], L.conv2d_dgrad(q(dz), q(w), xin.shape, t.stride, t.pad))
        elif t.kind == "lrn":
            acc(t.inputs[0], L.lrn_bwd(dy, get(t.inputs[0])))
        elif t.kind == "fc_relu_drop":
            xf, z, keep = caches[i]
            dxf, dw, db = L.fc_relu_dropout_bwd(q(dy[:, :, 0, 0]), q(xf), q(P[t.name + ".w"]), z, keep, t.ratio)
            grads[t.name + ".w"] += dw
            grads[t.name + ".b"] += db
            src = get(t.inputs[0])
            n, c, h, w = src.shape
            acc(t.inputs[0], dxf.reshape(n, h, w, c).transpose(0, 3, 1, 2))
        elif t.kind == "avgpool":
            acc(t.inputs[0], L.avgpool_bwd(dy[:, :, 0, 0], get(t.inputs[0]).shape))
    if map_grads is not None:
        map_grads.extend(gmap)
    return loss, grads, outs


def init_params(net: Net, seed: int = 2, bn_random: bool = False, residual_gamma=None) -> dict:
    """Seeded fp32 parameters (synthdata recipe). With ``bn_random`` gamma ~
    U(0.5,1.5), beta ~ U(-0.2,0.2) (parity tests, so gamma/beta mix-ups show).
    ``residual_gamma=(lo, hi)`` draws the last BN gamma of every residual branch
    (``gamma3``) from U(lo, hi) -- the small-residual initialisation of
    large-batch ResNet training (DESIGN.md Reading 28)."""
    g = synthdata.rng(seed)
    params = {}
    for name, shape in param_shapes(net).items():
        if name.endswith(".w"):
            fan_in = int(np.prod(shape[1:]))
            params[name] = synthdata.he_normal(shape, fan_in, g)
        elif name.endswith(".b"):
            params[name] = np.zeros(shape, np.float32)
        elif ".gamma" in name:
            params[name] = (g.uniform(0.5, 1.5, shape).astype(np.float32) if bn_random
                            else np.ones(shape, np.float32))
            if residual_gamma is not None and name.endswith(".gamma3"):
                params[name] = g.uniform(residual_gamma[0], residual_gamma[1], shape).astype(np.float32)
        else:
            params[name] = (g.uniform(-0.2, 0.2, shape).astype(np.float32) if bn_random
                            else np.zeros(shape, np.float32))
    return params


def sgd_step(params, moms, grads, lr, grad_scale=1.0):
    """Momentum SGD over every parameter."""
    newp, newm = {}, {}
    for k in params:
        newp[k], newm[k] = L.sgd_momentum(np.asarray(params[k], np.float64),
                                          np.asarray(moms[k], np.float64),
                                          grads[k], lr, grad_scale=grad_scale)
    return newp, newm
