// Plain, slow CPU C++ oracle of one verify step (BASELINE.json north_star: "a plain, slow CPU C++
// implementation sharing no code with the GPU path").  TEST INFRASTRUCTURE ONLY: loaded by
// tests/ (pinned against the numpy oracle, tests/test_oracle_cpp.py) and by bench.py's
// cpu_baseline / --impl reference legs; the product library never includes, links or calls it.
//
// It restates, line by line, the numpy oracle (oracle/model.py, oracle/verify.py,
// oracle/numerics.py), which follows the paper: the server "verifies [the draft tokens] in a single
// forward pass" and "returns both the verified tokens and one additional token" (PAPER.md P:171-173,
// §4.1) with per-sequence masks (§4.3):
//   O1 weights  : Philox4x32-10, bf16(f32(f32(int24) * scale))
//   O2 forward  : slot 0 = root at position L, node i at L + depth(i); per layer h = bf16(rmsnorm),
//                 q/k = f16(rope(h W^T)), v = f16(h W^T), attention over prefix + root +
//                 ancestors-or-self with the fp16 softmax numerator (DESIGN R-precision),
//                 O = bf16(o), x += O Wo^T, h2 = bf16(rmsnorm), M = bf16(silu(h2 Wg^T) * h2 Wu^T),
//                 x += M Wd^T; final hidden = rmsnorm (unrounded), logits = hf Wlm^T (float64)
//   O3 targets  : greedy argmax (ties -> lowest id) or Gumbel-max l/T + g (amb. A9)
//   O4 walk     : descend while a child carries the parent's target; bonus = the stop slot's target
// Arithmetic is float64 throughout, loops are plain (OpenMP over output features / slots only).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#include <omp.h>

namespace {

struct U4 { uint32_t x, y, z, w; };

U4 philox(U4 c, uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
  }
  return c;
}
uint32_t word_of(const U4& r, int i) { return i == 0 ? r.x : (i == 1 ? r.y : (i == 2 ? r.z : r.w)); }

// round-to-nearest-even onto a grid of `bits` significant bits with minimum exponent emin
double round_bits(double x, int bits, int emin, double overflow) {
  if (!std::isfinite(x)) return x;
  int e;
  std::frexp(x, &e);
  e = std::max(e - bits, emin);
  const double sp = std::ldexp(1.0, e);
  const double y = std::nearbyint(x / sp) * sp;
  if (std::fabs(y) >= overflow) return std::copysign(INFINITY, x);
  return y;
}
double bf16r(double x) { return round_bits(x, 8, -133, std::ldexp(1.0, 128)); }
double f16r(double x) { return round_bits(x, 11, -24, 65520.0); }
double bf16_bits(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return (double)f;
}
uint16_t to_bf16_bits(float v) {   // v is already exactly a bf16 value after bf16r
  uint32_t u;
  std::memcpy(&u, &v, 4);
  return (uint16_t)(u >> 16);
}

constexpr uint32_t kWeightTag = 0x57454947u;   // 'WEIG'
constexpr uint32_t kKvTag = 0x4B564649u;       // 'KVFI'
enum { T_EMBED = 1, T_WQ, T_WK, T_WV, T_WO, T_WG, T_WU, T_WD, T_LM, T_GATTN, T_GMLP, T_GFINAL };

}  // namespace

extern "C" {

struct oref_shape {
  int n_layers, d, n_heads, n_kv, head_dim, ffn, vocab;
  double eps, rope_theta;
};

struct oref_model {
  oref_shape s;
  uint64_t seed;
  std::vector<uint16_t> embed, lm;                      // [V][d]
  std::vector<std::vector<uint16_t>> wq, wk, wv, wo, wg, wu, wd;
  std::vector<std::vector<double>> g_attn, g_mlp;
  std::vector<double> g_final;
};

// O1: element idx of the logical row-major [rows][cols] matrix of tensor t, layer l
static void gen_matrix(std::vector<uint16_t>& out, uint64_t seed, int t, int l, long long rows, long long cols,
                       double stdv) {
  out.resize((size_t)(rows * cols));
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const float scale = (float)(stdv * std::sqrt(3.0) * std::ldexp(1.0, -23));
  const long long n4 = (rows * cols + 3) / 4;
#pragma omp parallel for schedule(static)
  for (long long q = 0; q < n4; ++q) {
    const U4 r = philox(U4{(uint32_t)q, (uint32_t)t, (uint32_t)l, kWeightTag}, k0, k1);
    for (int i = 0; i < 4 && 4 * q + i < rows * cols; ++i) {
      const int32_t i24 = (int32_t)(word_of(r, i) >> 8) - (1 << 23);
      const float v = (float)i24 * scale;
      out[(size_t)(4 * q + i)] = to_bf16_bits((float)bf16r((double)v));
    }
  }
}
static std::vector<double> gen_gain(uint64_t seed, int t, int l, int d) {
  std::vector<double> g(d);
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int i = 0; i < d; ++i) {
    const U4 r = philox(U4{(uint32_t)(i >> 2), (uint32_t)t, (uint32_t)l, kWeightTag}, k0, k1);
    const int32_t i24 = (int32_t)(word_of(r, i & 3) >> 8) - (1 << 23);
    const float v = (float)i24 * (float)std::ldexp(1.0, -25) + 1.0f;
    g[i] = bf16r((double)v);
  }
  return g;
}

// Weights of all layers and the LM head (bf16 bits); generation is setup, never timed.
oref_model* oref_model_create(const oref_shape* s, uint64_t seed) {
  oref_model* m = new oref_model();
  m->s = *s;
  m->seed = seed;
  const long long d = s->d, qd = (long long)s->n_heads * s->head_dim, kd = (long long)s->n_kv * s->head_dim,
                  F = s->ffn, V = s->vocab;
  gen_matrix(m->embed, seed, T_EMBED, 0, V, d, 1.0);
  gen_matrix(m->lm, seed, T_LM, 0, V, d, 2.0 / std::sqrt((double)d));
  const int L = s->n_layers;
  m->wq.resize(L); m->wk.resize(L); m->wv.resize(L); m->wo.resize(L); m->wg.resize(L); m->wu.resize(L); m->wd.resize(L);
  for (int l = 0; l < L; ++l) {
    gen_matrix(m->wq[l], seed, T_WQ, l, qd, d, 1.0 / std::sqrt((double)d));
    gen_matrix(m->wk[l], seed, T_WK, l, kd, d, 1.0 / std::sqrt((double)d));
    gen_matrix(m->wv[l], seed, T_WV, l, kd, d, 1.0 / std::sqrt((double)d));
    gen_matrix(m->wo[l], seed, T_WO, l, d, qd, 1.0 / std::sqrt((double)qd));
    gen_matrix(m->wg[l], seed, T_WG, l, F, d, 1.0 / std::sqrt((double)d));
    gen_matrix(m->wu[l], seed, T_WU, l, F, d, 1.0 / std::sqrt((double)d));
    gen_matrix(m->wd[l], seed, T_WD, l, d, F, 1.0 / std::sqrt((double)F));
    m->g_attn.push_back(gen_gain(seed, T_GATTN, l, s->d));
    m->g_mlp.push_back(gen_gain(seed, T_GMLP, l, s->d));
  }
  m->g_final = gen_gain(seed, T_GFINAL, 0, s->d);
  return m;
}
void oref_model_destroy(oref_model* m) { delete m; }

// Synthetic cached K or V (oracle/model.py gen_kv_fill): element e of token t
// = f16(f32(int24 * 2^-23)), Philox counter (e >> 2, t, layer*2 + kv_sel, stream ^ 'KVFI').
static void kv_fill(std::vector<double>& out, uint64_t seed, uint32_t stream, int layer, int kv_sel, int n_tok,
                    int per_tok) {
  out.resize((size_t)n_tok * per_tok);
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma omp parallel for schedule(static)
  for (int t = 0; t < n_tok; ++t)
    for (int q = 0; q < per_tok / 4; ++q) {
      const U4 r = philox(U4{(uint32_t)q, (uint32_t)t, (uint32_t)((layer << 1) | kv_sel), stream ^ kKvTag}, k0, k1);
      for (int i = 0; i < 4; ++i) {
        const int32_t i24 = (int32_t)(word_of(r, i) >> 8) - (1 << 23);
        out[(size_t)t * per_tok + 4 * q + i] = f16r((double)((float)i24 * (float)std::ldexp(1.0, -23)));
      }
    }
}

// y[s][f] = sum_i x[s][i] * W[f][i] (W: bf16 bits [nf][k]); four slots per pass over a weight row
static void matmul(const std::vector<double>& x, int S, int k, const std::vector<uint16_t>& W, int nf,
                   std::vector<double>& y) {
  y.assign((size_t)S * nf, 0.0);
#pragma omp parallel
  {
    std::vector<double> w(k);
#pragma omp for schedule(static)
    for (int f = 0; f < nf; ++f) {
      for (int i = 0; i < k; ++i) w[i] = bf16_bits(W[(size_t)f * k + i]);
      int s = 0;
      for (; s + 4 <= S; s += 4) {
        double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        const double *x0 = &x[(size_t)s * k], *x1 = x0 + k, *x2 = x1 + k, *x3 = x2 + k;
        for (int i = 0; i < k; ++i) {
          a0 += x0[i] * w[i];
          a1 += x1[i] * w[i];
          a2 += x2[i] * w[i];
          a3 += x3[i] * w[i];
        }
        y[(size_t)s * nf + f] = a0; y[(size_t)(s + 1) * nf + f] = a1;
        y[(size_t)(s + 2) * nf + f] = a2; y[(size_t)(s + 3) * nf + f] = a3;
      }
      for (; s < S; ++s) {
        double a = 0;
        const double* xs = &x[(size_t)s * k];
        for (int i = 0; i < k; ++i) a += xs[i] * w[i];
        y[(size_t)s * nf + f] = a;
      }
    }
  }
}

static void rmsnorm(const double* x, const std::vector<double>& g, int d, double eps, double* out) {
  double ss = 0;
  for (int i = 0; i < d; ++i) ss += x[i] * x[i];
  const double r = std::sqrt(ss / d + eps);
  for (int i = 0; i < d; ++i) out[i] = x[i] / r * g[i];
}

// Verify one request (O2-O4).  cache_k / cache_v: [layers][L][n_kv][hd] float64 of fp16 values, or
// null to use the synthetic fill (fill_seed, fill_stream).  mode 0 greedy, 1 Gumbel-max at T.
// Outputs: row_target / row_score [S = n + 1], logits [S][V] (nullable), accepted (len, tokens,
// nodes), bonus.  Returns 0, or -1 on an invalid tree (parent not in {-1} U [0, i)).
int oref_verify(const oref_model* m, int L, const double* cache_k, const double* cache_v, uint64_t fill_seed,
                uint32_t fill_stream, int root, int n, const int* parent, const int* token, int mode, double temperature,
                uint64_t seed, uint32_t round, uint64_t session, int* row_target, double* row_score, double* logits,
                int* acc_len, int* acc_tok, int* acc_node, int* bonus) {
  const oref_shape& s = m->s;
  const int S = n + 1, d = s.d, H = s.n_heads, KV = s.n_kv, hd = s.head_dim, G = H / KV, F = s.ffn, V = s.vocab;
  for (int i = 0; i < n; ++i)
    if (!(parent[i] == -1 || (parent[i] >= 0 && parent[i] < i))) return -1;
  // depth, RoPE positions, visible tree slots (root + ancestors-or-self, ascending)
  std::vector<int> depth(n);
  std::vector<std::vector<int>> vis(S);
  vis[0] = {0};
  for (int i = 0; i < n; ++i) {
    depth[i] = parent[i] < 0 ? 1 : depth[parent[i]] + 1;
    vis[i + 1] = vis[parent[i] < 0 ? 0 : parent[i] + 1];
    vis[i + 1].push_back(i + 1);
  }
  std::vector<double> pos(S);
  pos[0] = L;
  for (int i = 0; i < n; ++i) pos[i + 1] = L + depth[i];
  // residual stream x [S][d] = embeddings of root, node tokens
  std::vector<double> x((size_t)S * d), h((size_t)S * d), q, k, v, tmp;
  for (int sl = 0; sl < S; ++sl) {
    const int tok = sl == 0 ? root : token[sl - 1];
    for (int i = 0; i < d; ++i) x[(size_t)sl * d + i] = bf16_bits(m->embed[(size_t)tok * d + i]);
  }
  std::vector<double> inv_freq(hd / 2);
  for (int i = 0; i < hd / 2; ++i) inv_freq[i] = std::pow(s.rope_theta, -2.0 * (double)i / (double)hd);
  auto rope = [&](double* vec, double p) {   // rotate-half, one head
    for (int i = 0; i < hd / 2; ++i) {
      const double a = p * inv_freq[i], c = std::cos(a), sn = std::sin(a);
      const double x1 = vec[i], x2 = vec[i + hd / 2];
      vec[i] = x1 * c - x2 * sn;
      vec[i + hd / 2] = x2 * c + x1 * sn;
    }
  };
  std::vector<double> ck, cv, o((size_t)S * H * hd), ob, mg, mu, hm;
  for (int l = 0; l < s.n_layers; ++l) {
    for (int sl = 0; sl < S; ++sl) {
      rmsnorm(&x[(size_t)sl * d], m->g_attn[l], d, s.eps, &h[(size_t)sl * d]);
      for (int i = 0; i < d; ++i) h[(size_t)sl * d + i] = bf16r(h[(size_t)sl * d + i]);
    }
    matmul(h, S, d, m->wq[l], H * hd, q);
    matmul(h, S, d, m->wk[l], KV * hd, k);
    matmul(h, S, d, m->wv[l], KV * hd, v);
    for (int sl = 0; sl < S; ++sl) {
      for (int hh = 0; hh < H; ++hh) {
        double* qv = &q[((size_t)sl * H + hh) * hd];
        rope(qv, pos[sl]);
        for (int e = 0; e < hd; ++e) qv[e] = f16r(qv[e]);
      }
      for (int g = 0; g < KV; ++g) {
        double* kv_ = &k[((size_t)sl * KV + g) * hd];
        rope(kv_, pos[sl]);
        for (int e = 0; e < hd; ++e) {
          kv_[e] = f16r(kv_[e]);
          v[((size_t)sl * KV + g) * hd + e] = f16r(v[((size_t)sl * KV + g) * hd + e]);
        }
      }
    }
    const double* pk;
    const double* pv;
    if (cache_k) {
      pk = cache_k + (size_t)l * L * KV * hd;
      pv = cache_v + (size_t)l * L * KV * hd;
    } else {
      kv_fill(ck, fill_seed, fill_stream, l, 0, L, KV * hd);
      kv_fill(cv, fill_seed, fill_stream, l, 1, L, KV * hd);
      pk = ck.data();
      pv = cv.data();
    }
    // attention: slot sl, head hh over prefix [0, L) then the visible tree slots, in that order
    const double sqrt_hd = std::sqrt((double)hd);
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int sl = 0; sl < S; ++sl)
      for (int hh = 0; hh < H; ++hh) {
        const int g = hh / G;
        const double* qv = &q[((size_t)sl * H + hh) * hd];
        const int nk = L + (int)vis[sl].size();
        std::vector<double> sc(nk);
        for (int j = 0; j < nk; ++j) {
          const double* kk = j < L ? pk + ((size_t)j * KV + g) * hd : &k[((size_t)vis[sl][j - L] * KV + g) * hd];
          double a = 0;
          for (int e = 0; e < hd; ++e) a += qv[e] * kk[e];
          sc[j] = a / sqrt_hd;   // numpy: (q . k) / sqrt(hd)
        }
        double mx = -INFINITY;
        for (int j = 0; j < nk; ++j) mx = std::max(mx, sc[j]);
        double den = 0;
        for (int j = 0; j < nk; ++j) {
          sc[j] = std::exp(sc[j] - mx);
          den += sc[j];
        }
        double* ov = &o[((size_t)sl * H + hh) * hd];
        for (int e = 0; e < hd; ++e) ov[e] = 0;
        for (int j = 0; j < nk; ++j) {
          const double w = f16r(sc[j]) / den;   // fp16 numerator, unrounded denominator
          const double* vv = j < L ? pv + ((size_t)j * KV + g) * hd : &v[((size_t)vis[sl][j - L] * KV + g) * hd];
          for (int e = 0; e < hd; ++e) ov[e] += w * vv[e];
        }
      }
    ob.resize(o.size());
    for (size_t i = 0; i < o.size(); ++i) ob[i] = bf16r(o[i]);
    matmul(ob, S, H * hd, m->wo[l], d, tmp);
    for (size_t i = 0; i < x.size(); ++i) x[i] += tmp[i];
    for (int sl = 0; sl < S; ++sl) {
      rmsnorm(&x[(size_t)sl * d], m->g_mlp[l], d, s.eps, &h[(size_t)sl * d]);
      for (int i = 0; i < d; ++i) h[(size_t)sl * d + i] = bf16r(h[(size_t)sl * d + i]);
    }
    matmul(h, S, d, m->wg[l], F, mg);
    matmul(h, S, d, m->wu[l], F, mu);
    hm.resize((size_t)S * F);
    for (size_t i = 0; i < hm.size(); ++i) hm[i] = bf16r(mg[i] / (1.0 + std::exp(-mg[i])) * mu[i]);
    matmul(hm, S, F, m->wd[l], d, tmp);
    for (size_t i = 0; i < x.size(); ++i) x[i] += tmp[i];
  }
  for (int sl = 0; sl < S; ++sl) rmsnorm(&x[(size_t)sl * d], m->g_final, d, s.eps, &h[(size_t)sl * d]);
  std::vector<double> lg;
  matmul(h, S, d, m->lm, V, lg);
  // O3: target per slot
  const uint32_t sk0 = (uint32_t)seed ^ round, sk1 = (uint32_t)(seed >> 32);
  const bool sample = mode == 1 && temperature >= 1e-6;
  const double invT = (double)(float)(1.0 / temperature);
  for (int sl = 0; sl < S; ++sl) {
    double best = -INFINITY;
    int bi = 0;
    for (int vv = 0; vv < V; ++vv) {
      double sc = lg[(size_t)sl * V + vv];
      if (logits) logits[(size_t)sl * V + vv] = sc;
      if (sample) {
        const U4 r = philox(U4{(uint32_t)(vv >> 2), (uint32_t)sl, (uint32_t)session, (uint32_t)(session >> 32)}, sk0, sk1);
        const double u = (double)((word_of(r, vv & 3) >> 8) | 1u) * std::ldexp(1.0, -24);
        sc = sc * invT - std::log(-std::log(u));
      }
      if (sc > best) { best = sc; bi = vv; }
    }
    row_target[sl] = bi;
    row_score[sl] = best;
  }
  // O4: walk
  int cur = -1, a = 0;
  for (;;) {
    const int want = row_target[cur < 0 ? 0 : cur + 1];
    int nxt = -1;
    for (int c = 0; c < n; ++c)
      if (parent[c] == cur && token[c] == want) { nxt = c; break; }
    if (nxt < 0) break;
    acc_tok[a] = token[nxt];
    acc_node[a] = nxt;
    ++a;
    cur = nxt;
  }
  *acc_len = a;
  *bonus = row_target[cur < 0 ? 0 : cur + 1];
  return 0;
}

int oref_threads(void) { return omp_get_max_threads(); }

}  // extern "C"
