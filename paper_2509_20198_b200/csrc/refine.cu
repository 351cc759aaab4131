// K3: refiner CNN -- weight bundle, execution plan and refine epilogue.
//
//   ts_weights_create  <- load_weights + ArchDescriptor.from_text/validate +
//                         WeightBundle.validate (refiner.py:92-311)
//   ts_refine          <- refine_batch (refiner.py:475-528) / _Forward.run
//                         (refiner.py:430-441)
//   ts_conv2d          <- conv2d / _conv_batched (refiner.py:330-388)
//
// The topology is the reference's fixed one (4 encoders -> concat -> merge
// -> two decoders -> concat with the 8 raw input channels -> fuse -> crop);
// the descriptor fixes the layer sizes.  Activations are NHWC float32.
// Execution is crop-aware: the needed window of every layer is propagated
// backwards from the 64x64 crop, so decoder/fuse layers compute only the
// rows/columns that reach the crop (2.28 vs 3.59 GFLOP per tile for the
// default descriptor); results on the crop are unchanged.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "conv.cuh"
#include "tc_ptx.cuh"
#include "ts_common.cuh"

namespace ts {




namespace {

const char* kStages[8] = {"enc_hm_nn", "enc_hm_lin", "enc_rgb_nn", "enc_rgb_lin",
                          "merge", "dec_height", "dec_color", "fuse"};

struct LayerDesc {
  bool up2 = false;
  int ci = 0, co = 0, k = 0, s = 1, p = 0;
  bool lrelu = false;
};

struct Win {
  int y0, y1, x0, x1;
};

struct ConvLayer {
  int stage;            // index into kStages
  int index;            // position inside the stage's layer list
  bool up2;             // preceded by an Upsample2
  LayerDesc d;
  int Hin, Win_, Hout, Wout;  // physical input dims, output dims
  Win out_win;
  float* w = nullptr;   // device [K][Cout]
  float* b = nullptr;   // device [Cout]
  const uint8_t* w_tc = nullptr;  // tensor-core packed weights (or null)
  int w_layout = 0;               // which TC kernel the packed weights serve
  size_t out_off = 0;   // workspace offset (floats) of the output buffer
  int out_cstride = 0, out_coff = 0;
  int in_src = -1;      // -1: external/concat buffers handled by the planner
  // space-to-depth execution of a stride-2 3x3 layer (conv.cuh ActView):
  // s2d_in runs it as a stride-1 2x2 conv over 4*C_in channels (weights
  // remapped, dexec); s2d_out = this layer writes its output in that layout
  bool s2d_in = false, s2d_out = false;
  LayerDesc dexec;      // executed shape (== d unless s2d_in)
  // phase form of an up2 + 3x3 layer (conv.cuh ConvOp::ph): four 2x2
  // convolutions over the low-resolution input, one per output phase
  bool poly = false;
  const uint8_t* w_ph[4] = {nullptr, nullptr, nullptr, nullptr};
  Win ph_win[4];
  std::vector<float> w_host, b_host;  // final-layer kernel: weights as parameters
  bool h2 = false;          // executed on the wide-M halo kernel (or phases)
  int prec = 0;             // tensor-core precision mode of this layer's launches
  bool out_planes = false;  // writes pre-split planes (conv.cuh ActView)
};

// low-resolution window of output phase p (0/1) of a high-res window
inline void phase_window(int lo, int hi, int p, int& a, int& b) {
  a = (lo - p + 1) >> 1;
  b = ((hi - 1 - p) >> 1) + 1;
  if (b < a) b = a;
}

}  // namespace
}  // namespace ts

struct ts_weights {
  bool identity = false;
  int precision = 0;
  int device = -1;  // the CUDA device its buffers live on
  std::vector<ts::ConvLayer> layers;
  // per-tile float counts of the planner's buffers
  size_t cat_floats = 0, fuse_in_floats = 0, per_tile_floats = 0;
  int enc_out_c = 0, dec_h_c = 0, dec_c_c = 0, fuse_in_c = 0;
  int enc_hw = 0;
  size_t cat_off = 0, fuse_in_off = 0;
  bool enc0_fused = false;  // the four encoders' first layers in one launch
  bool fuse_in_planes = false;  // fuse-input buffer (raw inputs + decoders)
  bool cat_planes = false;      // encoder concat buffer (merge input)
  int plane_fmt = 1;            // ActView planes format: 1 bf16, 2 FP16X3
  ts::Win fuse_in_win{0, 0, 0, 0};  // the part of it fuse.0 reads (crop-aware)
  std::vector<void*> device_allocs;
};

namespace ts {
namespace {

// Execution switches: alternative formulations kept for A/B measurement
// (DESIGN.md §2), read from the environment once per process.  Defaults
// are the measured-best configuration; every setting computes the same
// result within the stated tolerance (planes: bit-identical).
struct Switches {
  bool s2d = true;             // TS_S2D=0: stride-2 layers without space-to-depth
  bool poly = true;            // TS_POLY=0: decoders as plain up2 + 3x3
  bool enc0 = true;            // TS_ENC0=0: four first-layer launches
  bool final_cuda = true;      // TS_FINAL=0: fuse.2 on the tensor cores
  bool planes = false;         // TS_PLANES=1: pre-split activation storage
  bool branch_streams = true;  // TS_BRANCH_STREAMS=0: branches serialised
};
const Switches& switches() {
  static const Switches sw = [] {
    auto on = [](const char* name, bool dflt) {
      const char* e = getenv(name);
      return e ? e[0] == '1' : dflt;
    };
    Switches w;
    w.s2d = on("TS_S2D", true);
    w.poly = on("TS_POLY", true);
    w.enc0 = on("TS_ENC0", true);
    w.final_cuda = on("TS_FINAL", true);
    w.planes = on("TS_PLANES", false);
    w.branch_streams = on("TS_BRANCH_STREAMS", true);
    return w;
  }();
  return sw;
}

int parse_descriptor(const std::string& text, bool& identity,
                     std::map<std::string, std::vector<LayerDesc>>& stages,
                     long long& declared) {
  std::vector<std::string> lines;
  std::istringstream is(text);
  std::string ln;
  while (std::getline(is, ln)) {
    if (!ln.empty() && ln[0] == '#') continue;
    size_t a = ln.find_first_not_of(" \t\r\n");
    if (a == std::string::npos) continue;
    size_t b = ln.find_last_not_of(" \t\r\n");
    lines.push_back(ln.substr(a, b - a + 1));
  }
  if (lines.empty() || lines[0].rfind("arch ", 0) != 0) return TS_E_SHAPE;
  if (lines[0] != "arch 1") return TS_E_VERSION;
  identity = lines.size() > 1 && lines[1] == "identity";
  declared = -1;
  if (identity) return TS_OK;
  std::vector<LayerDesc>* cur = nullptr;
  bool pending_up = false;
  for (size_t i = 1; i < lines.size(); ++i) {
    std::istringstream ls(lines[i]);
    std::string kw;
    ls >> kw;
    if (kw == "params") {
      ls >> declared;
    } else if (kw == "stage") {
      std::string name;
      ls >> name;
      cur = &stages[name];
      pending_up = false;
    } else if (kw == "up2") {
      if (!cur || pending_up) return TS_E_SHAPE;
      pending_up = true;
    } else if (kw == "conv") {
      if (!cur) return TS_E_SHAPE;
      LayerDesc d;
      std::string act;
      ls >> d.ci >> d.co >> d.k >> d.s >> d.p >> act;
      if (ls.fail()) return TS_E_SHAPE;
      d.up2 = pending_up;
      d.lrelu = act == "lrelu";
      pending_up = false;
      cur->push_back(d);
    } else {
      return TS_E_SHAPE;
    }
  }
  if (pending_up) return TS_E_SHAPE;
  return TS_OK;
}

int conv_out(int n, const LayerDesc& d) {
  const int nl = d.up2 ? 2 * n : n;
  return (nl + 2 * d.p - d.k) / d.s + 1;
}

// input window needed (physical coords) for an output window
Win need_in(const Win& o, const LayerDesc& d, int Hin, int Win_) {
  const int Hl = d.up2 ? 2 * Hin : Hin, Wl = d.up2 ? 2 * Win_ : Win_;
  Win w;
  w.y0 = std::max(0, o.y0 * d.s - d.p);
  w.y1 = std::min(Hl, (o.y1 - 1) * d.s - d.p + d.k);
  w.x0 = std::max(0, o.x0 * d.s - d.p);
  w.x1 = std::min(Wl, (o.x1 - 1) * d.s - d.p + d.k);
  if (d.up2) {
    w.y0 >>= 1; w.x0 >>= 1;
    w.y1 = ((w.y1 - 1) >> 1) + 1;
    w.x1 = ((w.x1 - 1) >> 1) + 1;
  }
  return w;
}

Win unite(const Win& a, const Win& b) {
  return Win{std::min(a.y0, b.y0), std::max(a.y1, b.y1), std::min(a.x0, b.x0),
             std::max(a.x1, b.x1)};
}

// raw inputs -> channels [0, 8) of the fuse input, over the window
// [y0, y0 + wy) x [x0, x0 + wx) that fuse.0 reads
__global__ void copy_inputs_kernel(const float* __restrict__ in, int64_t n_win,
                                   float* __restrict__ out, int cstride, int planes,
                                   int y0, int x0, int wy, int wx) {
  // n_win < 2^31 (checked by the caller): 32-bit index math
  const uint32_t per = (uint32_t)(wy * wx);
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < (uint32_t)n_win;
       w += gridDim.x * blockDim.x) {
    const uint32_t b = w / per;
    const uint32_t r = w - b * per;
    const int64_t i = ((int64_t)b * kRes + y0 + r / wx) * kRes + x0 + r % wx;  // pixel
    float v[8];
    tcx::ld_v8(in + 8 * i, v);
    if (planes) {  // pre-split channels 0..7 of the fuse input
      tcx::store8_planes(out + (int64_t)cstride * i, cstride, 0, v, planes == 2);
    } else if (cstride % 8 == 0) {
      tcx::st_v8(out + (int64_t)cstride * i, v);
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) out[(int64_t)cstride * i + c] = v[c];
    }
  }
}

// Crop, denormalise, clamp and the non-finite fallback (refiner.py:491-527).
__global__ void __launch_bounds__(256)
refine_epilogue_kernel(const float* __restrict__ fused, int fcs, int identity,
                       const float* __restrict__ in, float* __restrict__ out,
                       uint8_t* __restrict__ nonfinite) {
  const int b = blockIdx.x;
  const float* F = fused + (int64_t)b * kRes * kRes * fcs;
  const float* I = in + (int64_t)b * kRes * kRes * 8;
  int bad = 0;
  if (!identity) {
    for (int i = threadIdx.x; i < kOut * kOut; i += blockDim.x) {
      const int y = i / kOut + kCrop, x = i % kOut + kCrop;
      const float* v = F + ((int64_t)y * kRes + x) * fcs;
      bad |= !(isfinite(v[0]) && isfinite(v[1]) && isfinite(v[2]) && isfinite(v[3]));
    }
  }
  bad = __syncthreads_or(bad);
  for (int i = threadIdx.x; i < kOut * kOut; i += blockDim.x) {
    const int y = i / kOut + kCrop, x = i % kOut + kCrop;
    const float* src = I + ((int64_t)y * kRes + x) * 8;
    float4 o;
    if (identity || bad) {
      o.x = src[1] * 480.0f;
      o.y = src[5]; o.z = src[6]; o.w = src[7];
      if (identity) {
        o.y = fminf(fmaxf(o.y, 0.f), 1.f);
        o.z = fminf(fmaxf(o.z, 0.f), 1.f);
        o.w = fminf(fmaxf(o.w, 0.f), 1.f);
      }
    } else {
      const float* v = F + ((int64_t)y * kRes + x) * fcs;
      o.x = v[0] * 480.0f;
      o.y = fminf(fmaxf(v[1], 0.f), 1.f);
      o.z = fminf(fmaxf(v[2], 0.f), 1.f);
      o.w = fminf(fmaxf(v[3], 0.f), 1.f);
    }
    reinterpret_cast<float4*>(out)[(int64_t)b * kOut * kOut + i] = o;
  }
  if (threadIdx.x == 0 && nonfinite) nonfinite[b] = (uint8_t)(bad && !identity);
}

struct Blob {
  const uint8_t* p;
  size_t n, off = 0;
  bool ok = true;
  template <typename T>
  T get() {
    T v{};
    if (off + sizeof(T) > n) { ok = false; return v; }
    memcpy(&v, p + off, sizeof(T));
    off += sizeof(T);
    return v;
  }
};

constexpr int kSubBatch = 1024;

int build_plan(ts_weights* W, std::map<std::string, std::vector<LayerDesc>>& st,
               std::map<std::string, std::pair<std::vector<int>, std::vector<float>>>& tensors) {
  for (const char* s : kStages)
    if (!st.count(s) || st[s].empty()) return TS_E_SHAPE;
  const int enc_in[4] = {1, 1, 3, 3};
  // spatial forward pass + channel checks (ArchDescriptor.validate)
  int enc_hw = -1, enc_c = 0;
  for (int e = 0; e < 4; ++e) {
    auto& L = st[kStages[e]];
    if (L[0].ci != enc_in[e]) return TS_E_SHAPE;
    int hw = kRes, c = enc_in[e];
    for (auto& d : L) {
      if (d.ci != c) return TS_E_SHAPE;
      hw = conv_out(hw, d);
      c = d.co;
    }
    if (enc_hw >= 0 && hw != enc_hw) return TS_E_SHAPE;
    enc_hw = hw;
    enc_c += c;
  }
  int hw = enc_hw, c = enc_c;
  for (auto& d : st["merge"]) {
    if (d.ci != c) return TS_E_SHAPE;
    hw = conv_out(hw, d);
    c = d.co;
  }
  const int merge_hw = hw, merge_c = c;
  int dec_c_out[2];
  for (int k = 0; k < 2; ++k) {
    int h2 = merge_hw, c2 = merge_c;
    for (auto& d : st[kStages[5 + k]]) {
      if (d.ci != c2) return TS_E_SHAPE;
      h2 = conv_out(h2, d);
      c2 = d.co;
    }
    if (h2 != kRes) return TS_E_SHAPE;
    dec_c_out[k] = c2;
  }
  const int fin = 8 + dec_c_out[0] + dec_c_out[1];
  c = fin;
  hw = kRes;
  for (auto& d : st["fuse"]) {
    if (d.ci != c) return TS_E_SHAPE;
    hw = conv_out(hw, d);
    c = d.co;
  }
  if (c != 4 || hw != kRes) return TS_E_SHAPE;
  W->enc_out_c = enc_c;
  W->dec_h_c = dec_c_out[0];
  W->dec_c_c = dec_c_out[1];
  W->fuse_in_c = fin;
  W->enc_hw = enc_hw;

  // ---- layers in execution order with physical dims ----
  std::vector<ConvLayer> layers;
  auto add_stage = [&](int s, int Hin) {
    int h = Hin, li = 0;
    for (auto& d : st[kStages[s]]) {
      if (d.up2) ++li;  // the Upsample2 entry occupies a layer index
      ConvLayer L;
      L.stage = s;
      L.index = li++;
      L.up2 = d.up2;
      L.d = d;
      L.Hin = h; L.Win_ = h;
      L.Hout = conv_out(h, d); L.Wout = L.Hout;
      h = L.Hout;
      layers.push_back(L);
    }
  };
  for (int s = 0; s < 4; ++s) add_stage(s, kRes);
  add_stage(4, enc_hw);
  add_stage(5, merge_hw);
  add_stage(6, merge_hw);
  add_stage(7, kRes);

  // ---- backward window propagation from the crop ----
  const int nL = (int)layers.size();
  std::vector<int> stage_first(8, -1), stage_last(8, -1);
  for (int i = 0; i < nL; ++i) {
    if (stage_first[layers[i].stage] < 0) stage_first[layers[i].stage] = i;
    stage_last[layers[i].stage] = i;
  }
  auto back = [&](int s, Win w) {  // returns needed window of the stage input
    for (int i = stage_last[s]; i >= stage_first[s]; --i) {
      if (layers[i].s2d_out) {  // s2d pixels are written whole (2x2 groups)
        w.y0 &= ~1; w.x0 &= ~1;
        w.y1 = std::min(layers[i].Hout, (w.y1 + 1) & ~1);
        w.x1 = std::min(layers[i].Wout, (w.x1 + 1) & ~1);
      }
      layers[i].out_win = w;
      w = need_in(w, layers[i].d, layers[i].Hin, layers[i].Win_);
    }
    return w;
  };
  Win crop{kCrop, kCrop + kOut, kCrop, kCrop + kOut};
  auto propagate = [&]() {
    const Win fuse_in_need = back(7, crop);
    W->fuse_in_win = fuse_in_need;
    Win merge_need = unite(back(5, fuse_in_need), back(6, fuse_in_need));
    Win enc_need = back(4, merge_need);
    for (int s = 0; s < 4; ++s) back(s, enc_need);
  };
  for (auto& L : layers) L.dexec = L.d;
  propagate();
  // stride-2 3x3 encoder layers run as stride-1 2x2 convolutions over a
  // space-to-depth input on the wide-M halo kernel (bf16 operand modes): a
  // strided im2col gather re-reads the input 9x and cannot use the halo
  // reuse.  The producing layer must be able to write s2d (direct kernel or
  // halo2), else the layer keeps its plain form.
  {
    const bool s2d_ok = tc16_mode(W->precision) && switches().s2d;
    auto exec_shape = [&](const ConvLayer& L, const LayerDesc& d) {
      ConvOp o{};
      o.k = d.k; o.stride = d.s; o.pad = d.p; o.up2 = L.up2;
      o.oy0 = L.out_win.y0; o.oy1 = L.out_win.y1; o.ox0 = L.out_win.x0; o.ox1 = L.out_win.x1;
      o.in.C = d.ci; o.in.cstride = d.ci; o.out.C = d.co; o.out.cstride = d.co;
      o.in.H = L.s2d_in ? L.Hin / 2 : L.Hin; o.in.W = o.in.H;
      o.batch = 1;
      return o;
    };
    for (int s = 0; s < 4 && s2d_ok; ++s)
      for (int i = stage_first[s] + 1; i <= stage_last[s]; ++i) {
        ConvLayer& L = layers[i];
        ConvLayer& P = layers[i - 1];
        const LayerDesc& d = L.d;
        if (d.s != 2 || d.k != 3 || d.p != 1 || L.up2 || L.Hin % 2 || L.Win_ % 2) continue;
        LayerDesc x = d;
        x.ci = 4 * d.ci; x.k = 2; x.s = 1; x.p = 1;
        L.s2d_in = true;
        const bool l_ok = conv_tc_halo2_eligible(exec_shape(L, x), W->precision);
        const ConvOp ps = exec_shape(P, P.dexec);
        const bool p_ok = P.s2d_in || (conv_direct_supported(ps) &&
                                       (P.dexec.ci <= 4 || P.dexec.co <= 16));
        if (!l_ok || !p_ok) { L.s2d_in = false; continue; }
        L.dexec = x;
        P.s2d_out = true;
      }
    propagate();
    bool ok = true;
    for (auto& L : layers)
      if (L.s2d_in && !conv_tc_halo2_eligible(exec_shape(L, L.dexec), W->precision)) ok = false;
    if (!ok) {
      for (auto& L : layers) { L.s2d_in = L.s2d_out = false; L.dexec = L.d; }
      propagate();
    }
  }

  // nearest-up2 + 3x3 layers (the decoders) run in phase form on the
  // wide-M halo kernel: 4/9 of the MACs, and the halo is gathered at the
  // input's own resolution
  {
    const bool poly_ok = tc16_mode(W->precision) && switches().poly;
    for (auto& L : layers) {
      const LayerDesc& d = L.d;
      if (!poly_ok || !L.up2 || d.k != 3 || d.s != 1 || d.p != 1 || L.s2d_in || L.s2d_out ||
          d.ci % 4)
        continue;
      bool ok = true;
      for (int p = 0; p < 4 && ok; ++p) {
        Win& w = L.ph_win[p];
        phase_window(L.out_win.y0, L.out_win.y1, p >> 1, w.y0, w.y1);
        phase_window(L.out_win.x0, L.out_win.x1, p & 1, w.x0, w.x1);
        ConvOp o{};
        o.k = 2; o.stride = 1; o.pad = 1; o.up2 = 0; o.ph = 1; o.ph_y = p >> 1; o.ph_x = p & 1;
        o.oy0 = w.y0; o.oy1 = w.y1; o.ox0 = w.x0; o.ox1 = w.x1;
        o.in.C = d.ci; o.in.cstride = d.ci; o.out.C = d.co; o.out.cstride = d.co;
        o.in.H = L.Hin; o.in.W = L.Win_;
        o.batch = 1;
        ok = conv_tc_halo2_eligible(o, W->precision);
      }
      L.poly = ok;
    }
  }

  // the four first encoder layers share one input read (conv_enc0.cu)
  {
    bool ok = switches().enc0 && tc16_mode(W->precision);
    const ConvLayer* f[4];
    for (int st = 0; st < 4 && ok; ++st) {
      f[st] = &layers[stage_first[st]];
      const ConvLayer& L = *f[st];
      ok = L.d.k == 3 && L.d.s == 2 && L.d.p == 1 && !L.up2 && L.s2d_out && !L.s2d_in &&
           L.Hin == kRes && L.d.co == f[0]->d.co && L.out_win.y0 == f[0]->out_win.y0 &&
           L.out_win.y1 == f[0]->out_win.y1 && L.out_win.x0 == f[0]->out_win.x0 &&
           L.out_win.x1 == f[0]->out_win.x1;
    }
    if (ok) {
      Enc0Op probe{};
      const int ch0[4] = {0, 1, 2, 5}, cin[4] = {1, 1, 3, 3};
      for (int st = 0; st < 4; ++st) { probe.ch0[st] = ch0[st]; probe.cin[st] = cin[st]; }
      probe.oy0 = f[0]->out_win.y0; probe.ox0 = f[0]->out_win.x0;
      ok = conv_enc0_supported(probe, f[0]->d.co);
    }
    W->enc0_fused = ok;
  }

  // ---- weights upload + buffer offsets (floats per tile) ----
  size_t off = 0;
  auto alloc = [&](size_t floats) {
    const size_t o = off;
    off += (floats + 63) & ~size_t(63);
    return o;
  };
  W->cat_off = alloc((size_t)enc_hw * enc_hw * enc_c);
  W->fuse_in_off = alloc((size_t)kRes * kRes * fin);
  int enc_coff = 0;
  size_t params = 0;
  for (int i = 0; i < nL; ++i) {
    ConvLayer& L = layers[i];
    const bool last = i == stage_last[L.stage];
    if (L.stage < 4 && last) {
      L.out_off = W->cat_off; L.out_cstride = enc_c; L.out_coff = enc_coff;
      enc_coff += L.d.co;
    } else if ((L.stage == 5 || L.stage == 6) && last) {
      L.out_off = W->fuse_in_off; L.out_cstride = fin;
      L.out_coff = L.stage == 5 ? 8 : 8 + dec_c_out[0];
    } else {
      L.out_off = alloc((size_t)L.Hout * L.Wout * L.d.co);
      L.out_cstride = L.d.co; L.out_coff = 0;
    }
    const std::string base = std::string(kStages[L.stage]) + "." + std::to_string(L.index);
    auto wi = tensors.find(base + ".weight");
    auto bi = tensors.find(base + ".bias");
    if (wi == tensors.end() || bi == tensors.end()) return TS_E_SHAPE;
    const auto& ws = wi->second.first;
    if (ws.size() != 4 || ws[0] != L.d.co || ws[1] != L.d.ci || ws[2] != L.d.k ||
        ws[3] != L.d.k)
      return TS_E_SHAPE;
    if (bi->second.first.size() != 1 || bi->second.first[0] != L.d.co) return TS_E_SHAPE;
    const LayerDesc& dx = L.dexec;
    const int K = dx.k * dx.k * dx.ci, Co = dx.co;
    std::vector<float> packed((size_t)K * Co);
    std::vector<float> src = wi->second.second;  // OIKK of the executed shape
    // FP16X3 layers run on the wide-M halo kernel with the accumulator
    // restarted and promoted to fp32 registers every <= 18 K steps
    // (tc_ptx.cuh Mode<5>)
    L.prec = W->precision;
    if (L.s2d_in) {
      // W'[o][(a*2+b)*ci + c][ty][tx] = W[o][c][2ty+a-1][2tx+b-1] (0 outside)
      const int ci0 = L.d.ci;
      std::vector<float> t((size_t)Co * dx.ci * 4, 0.f);
      for (int o = 0; o < Co; ++o)
        for (int a = 0; a < 2; ++a)
          for (int b = 0; b < 2; ++b)
            for (int c = 0; c < ci0; ++c)
              for (int ty = 0; ty < 2; ++ty)
                for (int tx = 0; tx < 2; ++tx) {
                  const int ky = 2 * ty + a - 1, kx = 2 * tx + b - 1;
                  if (ky < 0 || ky > 2 || kx < 0 || kx > 2) continue;
                  t[(((size_t)o * dx.ci + (a * 2 + b) * ci0 + c) * 2 + ty) * 2 + tx] =
                      src[(((size_t)o * ci0 + c) * 3 + ky) * 3 + kx];
                }
      src.swap(t);
    }
    for (int o = 0; o < Co; ++o)
      for (int ci = 0; ci < dx.ci; ++ci)
        for (int ky = 0; ky < dx.k; ++ky)
          for (int kx = 0; kx < dx.k; ++kx)
            packed[(size_t)((ky * dx.k + kx) * dx.ci + ci) * Co + o] =
                src[(((size_t)o * dx.ci + ci) * dx.k + ky) * dx.k + kx];
    params += packed.size() + Co;
    {  // the last layer (fuse.2 shape) runs on conv_final.cu when it fits
      ConvOp fs{};
      fs.k = dx.k; fs.stride = dx.s; fs.pad = dx.p; fs.up2 = L.up2;
      fs.in.C = dx.ci; fs.in.cstride = dx.ci; fs.out.C = Co; fs.out.cstride = Co;
      if (i == nL - 1 && conv_final_supported(fs) && switches().final_cuda) {
        L.w_host = packed;
        L.b_host = bi->second.second;
      }
    }
    TS_CUDA_TRY(cudaMalloc(&L.w, packed.size() * sizeof(float)));
    TS_CUDA_TRY(cudaMalloc(&L.b, Co * sizeof(float)));
    W->device_allocs.push_back(L.w);
    W->device_allocs.push_back(L.b);
    TS_CUDA_TRY(cudaMemcpy(L.w, packed.data(), packed.size() * sizeof(float),
                           cudaMemcpyHostToDevice));
    TS_CUDA_TRY(cudaMemcpy(L.b, bi->second.second.data(), Co * sizeof(float),
                           cudaMemcpyHostToDevice));
    if (L.poly) {
      for (int p = 0; p < 4; ++p) {
        // folded 2x2 weights of phase p: sums of the 3x3 taps each low-res
        // tap collects (fp64 sums rounded once)
        const int py = p >> 1, px = p & 1;
        std::vector<float> w2((size_t)Co * dx.ci * 4);
        for (int o = 0; o < Co; ++o)
          for (int ci = 0; ci < dx.ci; ++ci)
            for (int ty = 0; ty < 2; ++ty)
              for (int tx = 0; tx < 2; ++tx) {
                double acc = 0.0;
                for (int ky = 0; ky < 3; ++ky)
                  for (int kx = 0; kx < 3; ++kx)
                    if (phase_tap(py, ty, ky) && phase_tap(px, tx, kx))
                      acc += src[(((size_t)o * dx.ci + ci) * 3 + ky) * 3 + kx];
                w2[(((size_t)o * dx.ci + ci) * 2 + ty) * 2 + tx] = (float)acc;
              }
        ConvOp shape{};
        shape.k = 2; shape.stride = 1; shape.pad = 1; shape.ph = 1; shape.ph_y = py;
        shape.ph_x = px;
        shape.oy0 = L.ph_win[p].y0; shape.oy1 = L.ph_win[p].y1;
        shape.ox0 = L.ph_win[p].x0; shape.ox1 = L.ph_win[p].x1;
        shape.in.C = dx.ci; shape.in.cstride = dx.ci; shape.out.C = Co; shape.out.cstride = Co;
        shape.in.H = L.Hin; shape.in.W = L.Win_;
        shape.batch = 1;
        const std::vector<uint8_t> pk =
            pack_tc_weights_halo2(w2.data(), Co, dx.ci, 2, L.prec, shape);
        if (pk.empty()) return TS_E_INVALID;
        void* dp = nullptr;
        TS_CUDA_TRY(cudaMalloc(&dp, pk.size()));
        W->device_allocs.push_back(dp);
        TS_CUDA_TRY(cudaMemcpy(dp, pk.data(), pk.size(), cudaMemcpyHostToDevice));
        L.w_ph[p] = reinterpret_cast<const uint8_t*>(dp);
      }
    } else if (W->precision != 0 && dx.ci % 4 == 0) {
      ConvOp shape{};
      shape.k = dx.k;
      shape.stride = dx.s;
      shape.pad = dx.p;
      shape.up2 = L.up2;
      shape.oy0 = L.out_win.y0; shape.oy1 = L.out_win.y1;
      shape.ox0 = L.out_win.x0; shape.ox1 = L.out_win.x1;
      shape.in.C = dx.ci; shape.in.cstride = dx.ci; shape.out.C = Co;
      shape.out.cstride = Co;
      shape.in.H = L.s2d_in ? L.Hin / 2 : L.Hin; shape.in.W = shape.in.H;
      shape.batch = 1;
      L.w_layout = tc_weight_layout(shape, L.prec);
      const std::vector<uint8_t> pk =
          pack_tc_weights(src.data(), Co, dx.ci, dx.k, L.prec, shape, L.w_layout);
      if (L.s2d_in && L.w_layout != 2) return TS_E_INVALID;  // planner invariant
      void* d = nullptr;
      TS_CUDA_TRY(cudaMalloc(&d, pk.size()));
      W->device_allocs.push_back(d);
      TS_CUDA_TRY(cudaMemcpy(d, pk.data(), pk.size(), cudaMemcpyHostToDevice));
      L.w_tc = reinterpret_cast<const uint8_t*>(d);
    }
  }
  (void)params;
  if (tensors.size() != (size_t)nL * 2) return TS_E_SHAPE;  // unexpected tensors
  // Which layers run on the wide-M halo kernel (mirrors ts_refine's
  // dispatch), and which outputs are stored pre-split: those whose every
  // consumer is such a layer, so its producers only copy.
  for (auto& L : layers)
    L.h2 = L.poly || (L.w_tc && L.w_layout == 2 && L.dexec.ci > 4);
  {
    // Pre-split storage (TS_PLANES=1, opt-in): producing epilogues write
    // the consumer's operand planes (bf16 RN hi/lo, or the FP16X3 scaled
    // fp16 pair) and the halo producers only copy (cp.async for FP16X3).
    // Measured slower in every mode: bf16-class 12.96 vs 11.88 ms per 1,024
    // tiles, FP16X3 12.08 vs 10.04 ms (the epilogues' split and plane stores
    // cost more than the producers save; profiles/r02_cnn_layers.md).
    // Results are bit-identical either way.
    W->plane_fmt = W->precision == 5 ? 2 : 1;
    const bool on = tc16_mode(W->precision) && switches().planes;
    auto fmt_ok = [](const ConvLayer& L) {
      return L.d.co % 16 == 0 && L.out_cstride % 8 == 0 && L.out_coff % 8 == 0;
    };
    for (int i = 0; i < nL && on; ++i) {
      ConvLayer& L = layers[i];
      const bool last = i == stage_last[L.stage];
      bool all_h2 = false;
      if (!last) {
        all_h2 = layers[i + 1].h2 && layers[i + 1].dexec.ci % 8 == 0;
      } else if (L.stage == 4) {  // merge output -> both decoders' first layers
        const ConvLayer& a = layers[stage_first[5]];
        const ConvLayer& b = layers[stage_first[6]];
        all_h2 = a.h2 && b.h2 && a.dexec.ci % 8 == 0;
      } else if (L.stage < 4) {  // encoder output -> the concat -> merge.0
        const ConvLayer& m = layers[stage_first[4]];
        all_h2 = m.h2 && m.dexec.ci % 8 == 0;
      }
      // writers that can emit planes: halo2 / phase layers, the regular
      // tensor-core kernel, the fused first encoder layers
      const bool writer = L.h2 || (L.w_tc && L.w_layout == 0 && L.dexec.ci > 4) ||
                          (W->enc0_fused && L.stage < 4 && L.index == 0);
      L.out_planes = all_h2 && writer && fmt_ok(L);
    }
    // the concat is pre-split only if every encoder writes it so
    W->cat_planes = on;
    for (int st = 0; st < 4; ++st)
      W->cat_planes = W->cat_planes && layers[stage_last[st]].out_planes;
    for (int st = 0; st < 4; ++st) layers[stage_last[st]].out_planes = W->cat_planes;
    // fuse input: raw-input copy + both decoders' last layers -> fuse.0
    const ConvLayer& f0 = layers[stage_first[7]];
    W->fuse_in_planes = on && f0.h2 && fin % 8 == 0 && dec_c_out[0] % 16 == 0 &&
                        dec_c_out[1] % 16 == 0 && layers[stage_last[5]].h2 &&
                        layers[stage_last[6]].h2;
    layers[stage_last[5]].out_planes = W->fuse_in_planes;
    layers[stage_last[6]].out_planes = W->fuse_in_planes;
  }
  W->per_tile_floats = off;
  W->layers = std::move(layers);
  return TS_OK;
}

}  // namespace
}  // namespace ts

using namespace ts;

extern "C" int ts_weights_create(const uint8_t* lswb, size_t n_bytes, int precision,
                                 ts_weights** out) {
  if (!lswb || !out || precision < 0 || precision > 5) return TS_E_INVALID;
  *out = nullptr;
  if (n_bytes < 4 || memcmp(lswb, "LSWB", 4) != 0) return TS_E_BAD_MAGIC;
  Blob bl{lswb, n_bytes, 4};
  const uint32_t version = bl.get<uint32_t>();
  const uint32_t count = bl.get<uint32_t>();
  if (!bl.ok) return TS_E_SHAPE;
  if (version != 1) return TS_E_VERSION;
  std::map<std::string, std::pair<std::vector<int>, std::vector<float>>> tensors;
  for (uint32_t t = 0; t < count; ++t) {
    const uint16_t nl = bl.get<uint16_t>();
    if (!bl.ok || bl.off + nl > n_bytes) return TS_E_SHAPE;
    std::string name(reinterpret_cast<const char*>(lswb + bl.off), nl);
    bl.off += nl;
    const uint8_t rank = bl.get<uint8_t>();
    std::vector<int> dims(rank);
    size_t cnt = 1;
    for (int r = 0; r < rank; ++r) { dims[r] = (int)bl.get<uint32_t>(); cnt *= dims[r]; }
    if (!bl.ok || bl.off + 4 * cnt > n_bytes) return TS_E_SHAPE;
    std::vector<float> data(cnt);
    memcpy(data.data(), lswb + bl.off, 4 * cnt);
    bl.off += 4 * cnt;
    tensors[name] = {dims, std::move(data)};
  }
  const uint32_t dl = bl.get<uint32_t>();
  if (!bl.ok || bl.off + dl > n_bytes) return TS_E_SHAPE;
  std::string text(reinterpret_cast<const char*>(lswb + bl.off), dl);
  bool identity = false;
  long long declared = -1;
  std::map<std::string, std::vector<LayerDesc>> stages;
  int st = parse_descriptor(text, identity, stages, declared);
  if (st != TS_OK) return st;
  std::unique_ptr<ts_weights> W(new ts_weights());
  W->identity = identity;
  W->precision = precision;
  TS_CUDA_TRY(cudaGetDevice(&W->device));
  if (identity) {
    if (!tensors.empty()) return TS_E_SHAPE;
    *out = W.release();
    return TS_OK;
  }
  long long params = 0;
  for (auto& kv : stages)
    for (auto& d : kv.second) params += (long long)d.co * d.ci * d.k * d.k + d.co;
  if (declared >= 0 && declared != params) return TS_E_SHAPE;
  st = build_plan(W.get(), stages, tensors);
  if (st != TS_OK) {
    for (void* p : W->device_allocs) cudaFree(p);
    return st;
  }
  *out = W.release();
  return TS_OK;
}

extern "C" int ts_weights_destroy(ts_weights* w) {
  if (!w) return TS_OK;
  for (void* p : w->device_allocs) cudaFree(p);
  delete w;
  return TS_OK;
}

extern "C" int ts_weights_is_identity(const ts_weights* w) { return w && w->identity; }

extern "C" size_t ts_refine_workspace(const ts_weights* w, int batch) {
  if (!w || w->identity) return 256;
  const int sb = std::min(batch, kSubBatch);
  return (w->per_tile_floats * (size_t)std::max(sb, 1)) * sizeof(float) + 256;
}

namespace ts {
namespace {
// Independent branches of the network (the four encoders, the two
// decoders) run on forked streams so one branch's persistent-kernel tail
// is filled by the next branch's tiles.  Per host thread and device.
struct Branches {
  cudaStream_t side[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t fork = nullptr, join[3] = {nullptr, nullptr, nullptr};
  int device = -1;
};
int branches_for(Branches*& out) {
  thread_local Branches cache[8];
  int dev = 0;
  TS_CUDA_TRY(cudaGetDevice(&dev));
  Branches& b = cache[dev & 7];
  if (b.device != dev) {
    for (int i = 0; i < 3; ++i) {
      TS_CUDA_TRY(cudaStreamCreateWithFlags(&b.side[i], cudaStreamNonBlocking));
      TS_CUDA_TRY(cudaEventCreateWithFlags(&b.join[i], cudaEventDisableTiming));
    }
    TS_CUDA_TRY(cudaEventCreateWithFlags(&b.fork, cudaEventDisableTiming));
    b.device = dev;
  }
  out = &b;
  return TS_OK;
}
}  // namespace
}  // namespace ts

extern "C" int ts_refine(const ts_weights* W, const float* d_in, int batch, float* d_out,
                         uint8_t* d_nonfinite, void* d_workspace, void* stream) {
  if (!W || batch < 0) return TS_E_INVALID;
  if (batch == 0) return TS_E_SHAPE;  // refine_batch requires a non-empty batch
  {
    int dev = -1;
    TS_CUDA_TRY(cudaGetDevice(&dev));
    if (dev != W->device) return TS_E_INVALID;  // handle built on another device
  }
  cudaStream_t s = as_stream(stream);
  if (W->identity) {
    ts::count_launch(), refine_epilogue_kernel<<<batch, 256, 0, s>>>(d_in, 8, 1, d_in, d_out, d_nonfinite);
    TS_LAUNCH_CHECK();
    return TS_OK;
  }
  float* ws = reinterpret_cast<float*>(d_workspace);
  const int fcs = W->layers.back().d.co;
  Branches* br = nullptr;
  {
    if (switches().branch_streams) {
      const int st = branches_for(br);
      if (st != TS_OK) return st;
    }
  }
  // region 0: encoder branches (stages 0-3), region 1: decoders (5, 6)
  auto nside = [](int region) { return region == 0 ? 3 : 1; };
  auto fork = [&](int region) -> int {
    TS_CUDA_TRY(cudaEventRecord(br->fork, s));
    for (int k = 0; k < nside(region); ++k) TS_CUDA_TRY(cudaStreamWaitEvent(br->side[k], br->fork, 0));
    return TS_OK;
  };
  auto join = [&](int region) -> int {
    for (int k = 0; k < nside(region); ++k) {
      TS_CUDA_TRY(cudaEventRecord(br->join[k], br->side[k]));
      TS_CUDA_TRY(cudaStreamWaitEvent(s, br->join[k], 0));
    }
    return TS_OK;
  };
  for (int b0 = 0; b0 < batch; b0 += kSubBatch) {
    const int B = std::min(kSubBatch, batch - b0);
    const float* in = d_in + (size_t)b0 * kRes * kRes * 8;
    auto buf = [&](size_t off) { return ws + off * B; };
    // raw inputs -> channels [0, 8) of the fuse input (skip concat); with
    // branch streams it runs beside the encoders (joined before the merge)
    bool copied = false;
    auto copy_inputs = [&](cudaStream_t cs) -> int {
      const Win& fw = W->fuse_in_win;
      const int wy = fw.y1 - fw.y0, wx = fw.x1 - fw.x0;
      const int64_t px = (int64_t)B * wy * wx;
      if (px >= (int64_t)INT32_MAX) return TS_E_INVALID;
      ts::count_launch(), copy_inputs_kernel<<<(int)std::min<int64_t>(ceil_div<int64_t>(px, 256), 148 * 16),
                           256, 0, cs>>>(in, px, buf(W->fuse_in_off), W->fuse_in_c,
                                         W->fuse_in_planes ? W->plane_fmt : 0, fw.y0, fw.x0, wy, wx);
      TS_LAUNCH_CHECK();
      copied = true;
      return TS_OK;
    };
    if (!br && copy_inputs(s) != TS_OK) return TS_E_CUDA;
    const int enc_ch0[4] = {0, 1, 2, 5};
    const int enc_cin[4] = {1, 1, 3, 3};
    const float* prev_base = nullptr;
    int prev_H = 0, prev_cs = 0, prev_coff = 0, prev_C = 0, prev_planes = 0;
    int prev_stage = -1;
    int region = -1;
    for (size_t i = 0; i < W->layers.size(); ++i) {
      const ConvLayer& L = W->layers[i];
      ConvOp op{};
      const bool first = (int)L.stage != prev_stage;
      void* lstream = stream;
      if (br) {
        const bool fused0 = W->enc0_fused && L.stage < 4 && L.index == 0;
        int want = region;
        if (!(fused0 && L.stage > 0))  // skipped fused layers keep the region
          want = (L.stage < 4 && !fused0) ? 0 : (L.stage == 5 || L.stage == 6) ? 1 : -1;
        if (want != region) {
          if (region >= 0 && join(region) != TS_OK) return TS_E_CUDA;
          if (want >= 0 && fork(want) != TS_OK) return TS_E_CUDA;
          if (want == 0 && !copied && copy_inputs(br->side[2]) != TS_OK) return TS_E_CUDA;
          region = want;
        }
        const int branch = region == 0 ? L.stage : region == 1 ? L.stage - 5 : 0;
        if (region >= 0 && branch > 0) lstream = br->side[branch - 1];
      }
      if (first) {
        if (L.stage < 4) {
          op.in = ActView{const_cast<float*>(in), kRes, kRes, 8, enc_ch0[L.stage],
                          enc_cin[L.stage]};
        } else if (L.stage == 4) {
          op.in = ActView{buf(W->cat_off), W->enc_hw, W->enc_hw, W->enc_out_c, 0,
                          W->enc_out_c, 0, W->cat_planes ? W->plane_fmt : 0};
        } else if (L.stage == 5 || L.stage == 6) {
          // merge output = the last merge layer's buffer
          size_t mi = 0;
          for (size_t j = 0; j < W->layers.size(); ++j)
            if (W->layers[j].stage == 4) mi = j;
          const ConvLayer& M = W->layers[mi];
          op.in = ActView{buf(M.out_off), M.Hout, M.Wout, M.out_cstride, M.out_coff, M.d.co,
                          0, M.out_planes ? W->plane_fmt : 0};
        } else {
          op.in = ActView{buf(W->fuse_in_off), kRes, kRes, W->fuse_in_c, 0, W->fuse_in_c,
                          0, W->fuse_in_planes ? W->plane_fmt : 0};
        }
      } else {
        op.in = ActView{const_cast<float*>(prev_base), prev_H, prev_H, prev_cs, prev_coff,
                        prev_C, 0, prev_planes};
      }
      if (L.s2d_in) {
        // previous layer wrote s2d: half-resolution pixels of 4 C channels
        if (prev_coff != 0 || prev_cs != prev_C) return TS_E_INVALID;
        op.in = ActView{const_cast<float*>(prev_base), prev_H / 2, prev_H / 2, 4 * prev_C, 0,
                        4 * prev_C, 0, prev_planes};
      }
      op.out = ActView{buf(L.out_off), L.Hout, L.Wout, L.out_cstride, L.out_coff, L.d.co, 0,
                       L.out_planes ? W->plane_fmt : 0};
      if (L.s2d_out) {
        if (L.out_coff != 0 || L.out_cstride != L.d.co) return TS_E_INVALID;
        op.out.cstride = 4 * L.d.co;
        op.out.s2d = 1;
      }
      op.up2 = L.up2;
      op.k = L.dexec.k; op.stride = L.dexec.s; op.pad = L.dexec.p;
      op.lrelu = L.d.lrelu;
      op.oy0 = L.out_win.y0; op.oy1 = L.out_win.y1;
      op.ox0 = L.out_win.x0; op.ox1 = L.out_win.x1;
      op.w = L.w; op.bias = L.b;
      op.batch = B;
      op.w_tc = L.w_tc;
      op.w_layout = L.w_layout;
      int st;
      if (W->enc0_fused && L.stage < 4 && L.index == 0) {
        if (L.stage == 0) {
          Enc0Op E{};
          E.in = in; E.H = kRes; E.W = kRes; E.batch = B;
          int e = 0;
          for (size_t j = 0; j < W->layers.size() && e < 4; ++j) {
            const ConvLayer& F = W->layers[j];
            if (F.stage != e || F.index != 0) continue;
            E.ch0[e] = enc_ch0[e]; E.cin[e] = enc_cin[e]; E.lrelu[e] = F.d.lrelu;
            E.w[e] = F.w; E.bias[e] = F.b;
            E.out[e] = ActView{buf(F.out_off), F.Hout, F.Wout, 4 * F.d.co, 0, F.d.co, 1,
                               F.out_planes ? W->plane_fmt : 0};
            ++e;
          }
          E.oy0 = L.out_win.y0; E.oy1 = L.out_win.y1; E.ox0 = L.out_win.x0; E.ox1 = L.out_win.x1;
          st = launch_conv_enc0(E, L.d.co, lstream);
          if (st != TS_OK) return st;
        }
        prev_base = buf(L.out_off); prev_H = L.Hout; prev_cs = L.out_cstride;
        prev_coff = L.out_coff; prev_C = L.d.co; prev_planes = L.out_planes ? W->plane_fmt : 0;
        prev_stage = L.stage;
        continue;
      }
      if (L.poly) {
        for (int p = 0; p < 4; ++p) {
          const Win& w = L.ph_win[p];
          if (w.y1 <= w.y0 || w.x1 <= w.x0) continue;
          ConvOp q = op;
          q.k = 2; q.stride = 1; q.pad = 1; q.up2 = 0;
          q.ph = 1; q.ph_y = p >> 1; q.ph_x = p & 1;
          q.oy0 = w.y0; q.oy1 = w.y1; q.ox0 = w.x0; q.ox1 = w.x1;
          q.w_tc = L.w_ph[p]; q.w_layout = 2;
          st = launch_conv_tc_halo2(q, L.prec, lstream);
          if (st != TS_OK) return st;
        }
        prev_base = op.out.base; prev_H = L.Hout; prev_cs = L.out_cstride;
        prev_coff = L.out_coff; prev_C = L.d.co; prev_planes = L.out_planes ? W->plane_fmt : 0;
        prev_stage = L.stage;
        continue;
      }
      // thin layers (few input or output channels: an MMA tile would be
      // mostly padding) -> fp32 direct kernel; the rest -> tensor cores (or
      // the fp32 CUDA-core GEMM in precision mode 0)
      if (!L.w_host.empty() && conv_final_supported(op)) {
        st = launch_conv_final(op, L.w_host.data(), L.b_host.data(), lstream);
        if (st != TS_OK) return st;
        prev_base = op.out.base; prev_H = L.Hout; prev_cs = L.out_cstride;
        prev_coff = L.out_coff; prev_C = L.d.co; prev_planes = L.out_planes ? W->plane_fmt : 0;
        prev_stage = L.stage;
        continue;
      }
      // (thin outputs with a wide input, e.g. fuse.2 32 -> 4, stay on the
      // wide-M halo kernel: N = 16 columns per plane, K = 9 x 32)
      const bool thin_tc = op.out.C <= 16 && op.in.C > 4 && L.w_tc && L.w_layout == 2 &&
                           !op.out.s2d;
      if (conv_direct_supported(op) && !thin_tc &&
          (op.in.C <= 4 || op.out.C <= 16 || W->precision == 0))
        st = launch_conv_direct(op, lstream);
      else if (L.w_tc && conv_tc_supported(op, L.prec))
        st = launch_conv_tc(op, L.prec, lstream);
      else
        st = launch_conv_simt(op, lstream);
      if (st != TS_OK) return st;
      prev_base = op.out.base; prev_H = L.Hout; prev_cs = L.out_cstride;
      prev_coff = L.out_coff; prev_C = L.d.co; prev_planes = L.out_planes ? W->plane_fmt : 0;
      prev_stage = L.stage;
    }
    if (br && region >= 0 && join(region) != TS_OK) return TS_E_CUDA;
    if (!copied) return TS_E_INVALID;  // every plan has an encoder region
    const ConvLayer& last = W->layers.back();
    ts::count_launch(), refine_epilogue_kernel<<<B, 256, 0, s>>>(buf(last.out_off), fcs, 0, in,
                                             d_out + (size_t)b0 * kOut * kOut * 4,
                                             d_nonfinite ? d_nonfinite + b0 : nullptr);
    TS_LAUNCH_CHECK();
  }
  return TS_OK;
}

namespace ts {
namespace {

__global__ void nchw_to_nhwc(const float* __restrict__ x, int B, int C, int H, int W,
                             float* __restrict__ y) {
  const int64_t n = (int64_t)B * C * H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % C, r = i / C;  // r = (b*H + y)*W + x
    const int64_t b = r / ((int64_t)H * W), yx = r % ((int64_t)H * W);
    y[i] = x[(b * C + c) * H * W + yx];
  }
}

__global__ void nhwc_to_nchw(const float* __restrict__ x, int B, int C, int H, int W,
                             float* __restrict__ y) {
  const int64_t n = (int64_t)B * C * H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t yx = i % ((int64_t)H * W), r = i / ((int64_t)H * W);
    const int64_t c = r % C, b = r / C;
    y[i] = x[(b * H * W + yx) * C + c];
  }
}

// OIKK -> [K][C_out] with K = (ky*k + kx)*C_in + ci
__global__ void pack_weights(const float* __restrict__ w, int Co, int Ci, int k,
                             float* __restrict__ out) {
  const int n = Co * Ci * k * k;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int kx = i % k, ky = (i / k) % k, ci = (i / (k * k)) % Ci, o = i / (k * k * Ci);
    out[(size_t)((ky * k + kx) * Ci + ci) * Co + o] = w[i];
  }
}

}  // namespace
}  // namespace ts

extern "C" int ts_conv2d(const float* d_x, int batch, int c_in, int h, int w,
                         const float* d_weight, int c_out, int k, const float* d_bias,
                         int stride, int padding, int precision, float* d_y,
                         void* stream) {
  if (batch <= 0 || c_in <= 0 || c_out <= 0 || k <= 0 || stride <= 0 || padding < 0)
    return TS_E_SHAPE;
  const int ho = (h + 2 * padding - k) / stride + 1;
  const int wo = (w + 2 * padding - k) / stride + 1;
  if (ho <= 0 || wo <= 0) return TS_E_SHAPE;
  cudaStream_t s = as_stream(stream);
  const size_t nin = (size_t)batch * c_in * h * w, nout = (size_t)batch * c_out * ho * wo;
  const size_t nw = (size_t)c_out * c_in * k * k;
  float* buf = nullptr;
  TS_CUDA_TRY(cudaMallocAsync(&buf, sizeof(float) * (nin + nout + nw), s));
  float *xin = buf, *yout = buf + nin, *wp = buf + nin + nout;
  const int g = 148 * 4;
  ts::count_launch(), nchw_to_nhwc<<<g, 256, 0, s>>>(d_x, batch, c_in, h, w, xin);
  ts::count_launch(), pack_weights<<<g, 256, 0, s>>>(d_weight, c_out, c_in, k, wp);
  ConvOp op{};
  op.in = ActView{xin, h, w, c_in, 0, c_in};
  op.out = ActView{yout, ho, wo, c_out, 0, c_out};
  op.up2 = 0; op.k = k; op.stride = stride; op.pad = padding; op.lrelu = 0;
  op.oy0 = 0; op.oy1 = ho; op.ox0 = 0; op.ox1 = wo;
  op.w = wp; op.bias = d_bias; op.batch = batch;
  int st;
  void* dpk = nullptr;
  if (precision != 0 && k * k * c_in > 0 && c_in % 4 == 0) {
    // tensor-core path: pack the swizzled weight images on the host
    std::vector<float> hw(nw);
    TS_CUDA_TRY(cudaMemcpyAsync(hw.data(), d_weight, nw * sizeof(float),
                                cudaMemcpyDeviceToHost, s));
    TS_CUDA_TRY(cudaStreamSynchronize(s));
    op.w_layout = tc_weight_layout(op, precision);
    const std::vector<uint8_t> pk =
        pack_tc_weights(hw.data(), c_out, c_in, k, precision, op, op.w_layout);
    TS_CUDA_TRY(cudaMallocAsync(&dpk, pk.size(), s));
    TS_CUDA_TRY(cudaMemcpyAsync(dpk, pk.data(), pk.size(), cudaMemcpyHostToDevice, s));
    op.w_tc = reinterpret_cast<const uint8_t*>(dpk);
    st = launch_conv_tc(op, precision, stream);
    TS_CUDA_TRY(cudaStreamSynchronize(s));  // pk (host) must outlive the copy
  } else {
    st = launch_conv_simt(op, stream);
  }
  if (dpk) TS_CUDA_TRY(cudaFreeAsync(dpk, s));
  if (st != TS_OK) return st;
  ts::count_launch(), nhwc_to_nchw<<<g, 256, 0, s>>>(yout, batch, c_out, ho, wo, d_y);
  TS_LAUNCH_CHECK();
  TS_CUDA_TRY(cudaFreeAsync(buf, s));
  return TS_OK;
}
