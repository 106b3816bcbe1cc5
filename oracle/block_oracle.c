/*
 * block_oracle.c — CPU fp32 restatement of the ISP transformer block, fwd + bwd.
 *
 * ORACLE / TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py as the checker. Never linked into the product.
 *
 * PARITY STATUS: activations/gradients are "parity unpinned" by the reference — the
 * reference (/root/reference/proj, seqplan) computes no tensors. This
 * file restates the block from the paper's prose and is cross-checked against an
 * independent PyTorch-autograd restatement (tests/test_oracle.py). Layout, schedule and
 * pool semantics ARE pinned to the reference (tests/test_seqplan_golden.py).
 *
 * Block ("Attention + MLP", 1732 SwiGLU 8/3, model.hpp:58-63
 * two norms, mempool.hpp:79-82 MLP width):
 *   n1 = RMSNorm(x) * g1 ; [q|k|v] = n1 Wqkv^T ; RoPE(q, k) (rotate-half, base 10000)
 *   o  = causal softmax(q k^T / sqrt(d)) v      (FlashAttention-fused MHA)
 *   h  = x + o Wo^T ; n2 = RMSNorm(h) * g2
 *   y  = h + (silu(n2 Wg^T) * (n2 Wu^T)) Wd^T
 * ISP sharding (cost.hpp:179-188): rank r owns tokens
 * [r S/p, (r+1) S/p) and the contiguous 1/p slice of every flattened weight
 * (ShardingLayout E/F, strategy.hpp:52-62); weights are all-gathered before use in fwd
 * and again in bwd, QKV and attention output pass through Ulysses all-to-alls (heads
 * [r D/p, (r+1) D/p) on rank r), weight gradients are reduce-scattered.
 *
 * Synthetic inputs are index-keyed: value = f(seed, tensor_id, flat_index)
 * via splitmix64 -> Box-Muller in double, so every rank's shard is identical for any p.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  int64_t H, D, S, I;
  double rope_base, eps;
} ob_shape;

enum { OB_NORM1 = 0, OB_QKV, OB_O, OB_NORM2, OB_GATE, OB_UP, OB_DOWN, OB_COUNT };

/* ------------------------------------------------------------------------------------
 * index-keyed synthetic data
 * ------------------------------------------------------------------------------------ */
static inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

double ob_keyed_normal(uint64_t seed, int tensor_id, int64_t idx) {
  const uint64_t base = splitmix64(seed * 0x9E3779B97F4A7C15ULL + (uint64_t)tensor_id);
  const uint64_t r1 = splitmix64(base ^ (uint64_t)(2 * idx));
  const uint64_t r2 = splitmix64(base ^ (uint64_t)(2 * idx + 1));
  const double u1 = (double)((r1 >> 11) + 1) * 0x1.0p-53; /* (0, 1] */
  const double u2 = (double)(r2 >> 11) * 0x1.0p-53;       /* [0, 1) */
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* out[i] = (float)(mean + std * N(seed, tid, offset + i)) */
void ob_fill(uint64_t seed, int tensor_id, int64_t offset, int64_t n, double mean, double stdv,
             float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    out[i] = (float)(mean + stdv * ob_keyed_normal(seed, tensor_id, offset + i));
}

/* RoPE table: cos/sin of t * base^(-2i/d), computed in double, stored fp32 [S, d/2]. */
void ob_rope_table(int64_t S, int64_t d, double base, float* cos_t, float* sin_t) {
  const int64_t half = d / 2;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < S; ++t)
    for (int64_t i = 0; i < half; ++i) {
      const double inv = pow(base, -2.0 * (double)i / (double)d);
      const double ang = (double)t * inv;
      cos_t[t * half + i] = (float)cos(ang);
      sin_t[t * half + i] = (float)sin(ang);
    }
}

/* ------------------------------------------------------------------------------------
 * dense kernels (row-major, fp32, OpenMP)
 * ------------------------------------------------------------------------------------ */
/* C[M,N] (+)= A[M,K] * B[N,K]^T, lda/ldb/ldc in elements */
static void mm_nt(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
                  int64_t ldb, float* C, int64_t ldc, int accumulate) {
#pragma omp parallel for schedule(static) collapse(2)
  for (int64_t i0 = 0; i0 < M; i0 += 16)
    for (int64_t j0 = 0; j0 < N; j0 += 16) {
      const int64_t i1 = i0 + 16 < M ? i0 + 16 : M;
      const int64_t j1 = j0 + 16 < N ? j0 + 16 : N;
      for (int64_t i = i0; i < i1; ++i)
        for (int64_t j = j0; j < j1; ++j) {
          const float* a = A + i * lda;
          const float* b = B + j * ldb;
          float acc[16] = {0};
          int64_t k = 0;
          for (; k + 16 <= K; k += 16)
            for (int l = 0; l < 16; ++l) acc[l] += a[k + l] * b[k + l];
          float s = 0.f;
          for (; k < K; ++k) s += a[k] * b[k];
          for (int l = 0; l < 16; ++l) s += acc[l];
          if (accumulate) C[i * ldc + j] += s;
          else C[i * ldc + j] = s;
        }
    }
}

/* C[M,N] (+)= A[M,K] * B[K,N]. Cache-blocked (16 rows x 512 columns of C per task, K in
 * blocks of 128 so the B block stays in L2 across the 16 rows); every C element still sums k
 * in ascending order, so the result is independent of the blocking. */
static void mm_nn(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
                  int64_t ldb, float* C, int64_t ldc, int accumulate) {
#pragma omp parallel for schedule(static) collapse(2)
  for (int64_t i0 = 0; i0 < M; i0 += 16)
    for (int64_t j0 = 0; j0 < N; j0 += 512) {
      const int64_t i1 = i0 + 16 < M ? i0 + 16 : M;
      const int64_t j1 = j0 + 512 < N ? j0 + 512 : N;
      if (!accumulate)
        for (int64_t i = i0; i < i1; ++i) memset(C + i * ldc + j0, 0, sizeof(float) * (size_t)(j1 - j0));
      for (int64_t k0 = 0; k0 < K; k0 += 128) {
        const int64_t k1 = k0 + 128 < K ? k0 + 128 : K;
        for (int64_t i = i0; i < i1; ++i) {
          float* c = C + i * ldc;
          for (int64_t k = k0; k < k1; ++k) {
            const float a = A[i * lda + k];
            const float* b = B + k * ldb;
            for (int64_t j = j0; j < j1; ++j) c[j] += a * b[j];
          }
        }
      }
    }
}

/* C[M,N] (+)= A[K,M]^T * B[K,N]  (weight gradients); blocked like mm_nn */
static void mm_tn(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
                  int64_t ldb, float* C, int64_t ldc, int accumulate) {
#pragma omp parallel for schedule(static) collapse(2)
  for (int64_t i0 = 0; i0 < M; i0 += 16)
    for (int64_t j0 = 0; j0 < N; j0 += 512) {
      const int64_t i1 = i0 + 16 < M ? i0 + 16 : M;
      const int64_t j1 = j0 + 512 < N ? j0 + 512 : N;
      if (!accumulate)
        for (int64_t i = i0; i < i1; ++i) memset(C + i * ldc + j0, 0, sizeof(float) * (size_t)(j1 - j0));
      for (int64_t k0 = 0; k0 < K; k0 += 128) {
        const int64_t k1 = k0 + 128 < K ? k0 + 128 : K;
        for (int64_t i = i0; i < i1; ++i) {
          float* c = C + i * ldc;
          for (int64_t k = k0; k < k1; ++k) {
            const float a = A[k * lda + i];
            const float* b = B + k * ldb;
            for (int64_t j = j0; j < j1; ++j) c[j] += a * b[j];
          }
        }
      }
    }
}

/* y = x * rstd * g ; rstd[t] saved */
static void rmsnorm_fwd(int64_t T, int64_t H, const float* x, const float* g, double eps,
                        float* y, float* rstd) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    const float* xr = x + t * H;
    double ss = 0;
    for (int64_t j = 0; j < H; ++j) ss += (double)xr[j] * xr[j];
    const float r = (float)(1.0 / sqrt(ss / (double)H + eps));
    rstd[t] = r;
    for (int64_t j = 0; j < H; ++j) y[t * H + j] = xr[j] * r * g[j];
  }
}

/* dx (+)= rstd*(dy*g - xhat*mean(dy*g*xhat)); dg_partial[j] += sum_t dy*xhat */
static void rmsnorm_bwd(int64_t T, int64_t H, const float* x, const float* g, const float* rstd,
                        const float* dy, float* dx, float* dg_partial) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    const float* xr = x + t * H;
    const float* dr = dy + t * H;
    const float r = rstd[t];
    double dot = 0;
    for (int64_t j = 0; j < H; ++j) dot += (double)dr[j] * g[j] * xr[j] * r;
    const float m = (float)(dot / (double)H);
    for (int64_t j = 0; j < H; ++j) dx[t * H + j] += r * (dr[j] * g[j] - xr[j] * r * m);
  }
  for (int64_t j = 0; j < H; ++j) {
    double s = 0;
    for (int64_t t = 0; t < T; ++t) s += (double)dy[t * H + j] * x[t * H + j] * rstd[t];
    dg_partial[j] += (float)s;
  }
}

/* rotate-half RoPE on q and k parts of qkv rows [T, 3H], global position t0 + t. dir=+1 fwd, -1 bwd */
static void rope_apply(int64_t T, int64_t t0, const ob_shape* sh, float* qkv, int64_t ld,
                       const float* cos_t, const float* sin_t, int dir) {
  const int64_t d = sh->H / sh->D, half = d / 2;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t)
    for (int part = 0; part < 2; ++part)
      for (int64_t h = 0; h < sh->D; ++h) {
        float* v = qkv + t * ld + part * sh->H + h * d;
        const float* c = cos_t + (t0 + t) * half;
        const float* s = sin_t + (t0 + t) * half;
        for (int64_t i = 0; i < half; ++i) {
          const float a = v[i], b = v[i + half];
          const float sn = dir > 0 ? s[i] : -s[i];
          v[i] = a * c[i] - b * sn;
          v[i + half] = b * c[i] + a * sn;
        }
      }
}

/* causal attention for heads [h0, h1) over all S tokens.
 * q,k,v,o: row t at base + t*ld, head h at column h*d. lse[(h-h0)*S + t]. */
static void attn_fwd(int64_t S, int64_t d, int64_t h0, int64_t h1, const float* q, const float* k,
                     const float* v, int64_t ld, float* o, int64_t ldo, float* lse) {
  const float scale = (float)(1.0 / sqrt((double)d));
#pragma omp parallel for schedule(dynamic, 8) collapse(2)
  for (int64_t h = h0; h < h1; ++h)
    for (int64_t t = 0; t < S; ++t) {
      float* p = (float*)malloc(sizeof(float) * (size_t)(t + 1));
      const float* qr = q + t * ld + h * d;
      float mx = -INFINITY;
      for (int64_t j = 0; j <= t; ++j) {
        const float* kr = k + j * ld + h * d;
        float s = 0;
        for (int64_t i = 0; i < d; ++i) s += qr[i] * kr[i];
        p[j] = s * scale;
        if (p[j] > mx) mx = p[j];
      }
      double sum = 0;
      for (int64_t j = 0; j <= t; ++j) {
        p[j] = expf(p[j] - mx);
        sum += p[j];
      }
      float* orow = o + t * ldo + h * d;
      for (int64_t i = 0; i < d; ++i) orow[i] = 0;
      for (int64_t j = 0; j <= t; ++j) {
        const float w = (float)(p[j] / sum);
        const float* vr = v + j * ld + h * d;
        for (int64_t i = 0; i < d; ++i) orow[i] += w * vr[i];
      }
      lse[(h - h0) * S + t] = mx + (float)log(sum);
      free(p);
    }
}

/* attention backward for heads [h0,h1); dq/dk/dv accumulate into zeroed buffers (ld). */
static void attn_bwd(int64_t S, int64_t d, int64_t h0, int64_t h1, const float* q, const float* k,
                     const float* v, int64_t ld, const float* o, const float* dout, int64_t ldo,
                     const float* lse, float* dq, float* dk, float* dv) {
  const float scale = (float)(1.0 / sqrt((double)d));
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t h = h0; h < h1; ++h) {
    float* P = (float*)malloc(sizeof(float) * (size_t)S);
    float* dS = (float*)malloc(sizeof(float) * (size_t)S);
    for (int64_t t = 0; t < S; ++t) {
      const float* qr = q + t * ld + h * d;
      const float* dor = dout + t * ldo + h * d;
      const float* orow = o + t * ldo + h * d;
      float Dt = 0;
      for (int64_t i = 0; i < d; ++i) Dt += dor[i] * orow[i];
      const float L = lse[(h - h0) * S + t];
      for (int64_t j = 0; j <= t; ++j) {
        const float* kr = k + j * ld + h * d;
        const float* vr = v + j * ld + h * d;
        float s = 0, dp = 0;
        for (int64_t i = 0; i < d; ++i) {
          s += qr[i] * kr[i];
          dp += dor[i] * vr[i];
        }
        P[j] = expf(s * scale - L);
        dS[j] = P[j] * (dp - Dt);
      }
      float* dqr = dq + t * ld + h * d;
      for (int64_t j = 0; j <= t; ++j) {
        const float* kr = k + j * ld + h * d;
        float* dkr = dk + j * ld + h * d;
        float* dvr = dv + j * ld + h * d;
        const float ds = dS[j] * scale;
        for (int64_t i = 0; i < d; ++i) {
          dqr[i] += ds * kr[i];
          dkr[i] += ds * qr[i];
          dvr[i] += P[j] * dor[i];
        }
      }
    }
    free(P);
    free(dS);
  }
}

static inline float silu_f(float x) { return x / (1.f + expf(-x)); }

/* ------------------------------------------------------------------------------------
 * per-rank state of the ISP-simulated executor (p = 1 is the unsharded block)
 * ------------------------------------------------------------------------------------ */
typedef struct {
  int64_t T, t0; /* local tokens and first global position */
  float *x, *n1, *r1, *qkv, *o_tok, *h, *n2, *r2, *g, *u, *a, *y;
  /* head-sharded attention operands: [S, 3*Hl] and [S, Hl] (Hl = H/p) */
  float *qkv_heads, *o_heads, *lse;
} ob_rank;

static float* zalloc(int64_t n) { return (float*)calloc((size_t)n, sizeof(float)); }

static void rank_alloc(ob_rank* R, const ob_shape* sh, int p, int r) {
  const int64_t H = sh->H, S = sh->S, I = sh->I, T = S / p, Hl = H / p;
  R->T = T;
  R->t0 = r * T;
  R->x = zalloc(T * H); R->n1 = zalloc(T * H); R->r1 = zalloc(T);
  R->qkv = zalloc(T * 3 * H); R->o_tok = zalloc(T * H); R->h = zalloc(T * H);
  R->n2 = zalloc(T * H); R->r2 = zalloc(T); R->g = zalloc(T * I); R->u = zalloc(T * I);
  R->a = zalloc(T * I); R->y = zalloc(T * H);
  R->qkv_heads = zalloc(S * 3 * Hl); R->o_heads = zalloc(S * Hl);
  R->lse = zalloc((sh->D / p) * S);
}

static void rank_free(ob_rank* R) {
  float* ps[] = {R->x, R->n1, R->r1, R->qkv, R->o_tok, R->h, R->n2, R->r2, R->g, R->u, R->a,
                 R->y, R->qkv_heads, R->o_heads, R->lse};
  for (size_t i = 0; i < sizeof(ps) / sizeof(ps[0]); ++i) free(ps[i]);
}

static int64_t tensor_numel(const ob_shape* sh, int t) {
  const int64_t H = sh->H, I = sh->I;
  switch (t) {
    case OB_NORM1: case OB_NORM2: return H;
    case OB_QKV: return 3 * H * H;
    case OB_O: return H * H;
    default: return I * H;
  }
}

/* Ulysses all-to-all, forward direction: token-sharded [T, 3H] on every rank ->
 * head-sharded [S, 3*Hl] (q|k|v blocks of Hl columns) on every rank. */
static void a2a_qkv_to_heads(const ob_shape* sh, int p, ob_rank* R) {
  const int64_t H = sh->H, Hl = H / p, T = sh->S / p;
  for (int dst = 0; dst < p; ++dst)
    for (int src = 0; src < p; ++src)
      for (int64_t t = 0; t < T; ++t)
        for (int part = 0; part < 3; ++part)
          memcpy(R[dst].qkv_heads + (src * T + t) * 3 * Hl + part * Hl,
                 R[src].qkv + t * 3 * H + part * H + dst * Hl, sizeof(float) * (size_t)Hl);
}
/* head-sharded [S, Hl] -> token-sharded [T, H] */
static void a2a_heads_to_tokens(const ob_shape* sh, int p, float* const* heads, int64_t ldh,
                                float* const* tok, int64_t ldt) {
  const int64_t H = sh->H, Hl = H / p, T = sh->S / p;
  for (int dst = 0; dst < p; ++dst)
    for (int src = 0; src < p; ++src)
      for (int64_t t = 0; t < T; ++t)
        memcpy(tok[dst] + t * ldt + src * Hl, heads[src] + (dst * T + t) * ldh,
               sizeof(float) * (size_t)Hl);
}
/* token-sharded [T, H] -> head-sharded [S, Hl] */
static void a2a_tokens_to_heads(const ob_shape* sh, int p, float* const* tok, int64_t ldt,
                                float* const* heads, int64_t ldh) {
  const int64_t H = sh->H, Hl = H / p, T = sh->S / p;
  for (int dst = 0; dst < p; ++dst)
    for (int src = 0; src < p; ++src)
      for (int64_t t = 0; t < T; ++t)
        memcpy(heads[dst] + (src * T + t) * ldh, tok[src] + t * ldt + dst * Hl,
               sizeof(float) * (size_t)Hl);
}

/*
 * ob_block_isp — the block on p simulated ranks (p = 1: unsharded).
 *   shards[t]   : concatenation over ranks of rank shards of tensor t (== full tensor,
 *                 flattened row-major; rank r owns [r E/p, (r+1) E/p))
 *   x, dy       : [S, H] (rank r owns rows [r S/p, (r+1) S/p))
 *   y, dx       : [S, H] outputs
 *   grad[t]     : full-size fp32 gradient, assembled from the per-rank reduce-scattered shards
 * Returns 0, or -1 on an unsupported shape.
 */
int ob_block_isp(const ob_shape* sh, int p, const float* const* shards, const float* x,
                 const float* dy, float* y, float* dx, float* const* grad) {
  const int64_t H = sh->H, D = sh->D, S = sh->S, I = sh->I, d = H / D;
  if (p < 1 || S % p || D % p || H % D || d % 2) return -1;
  const int64_t T = S / p, Hl = H / p, Dl = D / p;

  /* all-gather: concatenation of the contiguous shards is the full flattened tensor */
  float* W[OB_COUNT];
  for (int t = 0; t < OB_COUNT; ++t) {
    const int64_t n = tensor_numel(sh, t), per = n / p;
    W[t] = zalloc(n);
    for (int r = 0; r < p; ++r) memcpy(W[t] + r * per, shards[t] + r * per, sizeof(float) * (size_t)per);
  }
  float* cos_t = zalloc(S * (d / 2));
  float* sin_t = zalloc(S * (d / 2));
  ob_rope_table(S, d, sh->rope_base, cos_t, sin_t);

  ob_rank* R = (ob_rank*)calloc((size_t)p, sizeof(ob_rank));
  for (int r = 0; r < p; ++r) {
    rank_alloc(&R[r], sh, p, r);
    memcpy(R[r].x, x + r * T * H, sizeof(float) * (size_t)(T * H));
  }

  /* ---------------- forward ---------------- */
  for (int r = 0; r < p; ++r) {
    rmsnorm_fwd(T, H, R[r].x, W[OB_NORM1], sh->eps, R[r].n1, R[r].r1);
    mm_nt(T, 3 * H, H, R[r].n1, H, W[OB_QKV], H, R[r].qkv, 3 * H, 0);
    rope_apply(T, R[r].t0, sh, R[r].qkv, 3 * H, cos_t, sin_t, +1);
  }
  a2a_qkv_to_heads(sh, p, R);
  for (int r = 0; r < p; ++r) {
    float* qh = R[r].qkv_heads;
    /* local head j of rank r is global head r*Dl + j; operate on local column blocks */
    attn_fwd(S, d, 0, Dl, qh, qh + Hl, qh + 2 * Hl, 3 * Hl, R[r].o_heads, Hl, R[r].lse);
  }
  {
    float* heads[64];
    float* tok[64];
    for (int r = 0; r < p; ++r) { heads[r] = R[r].o_heads; tok[r] = R[r].o_tok; }
    a2a_heads_to_tokens(sh, p, heads, Hl, tok, H);
  }
  for (int r = 0; r < p; ++r) {
    ob_rank* Q = &R[r];
    mm_nt(T, H, H, Q->o_tok, H, W[OB_O], H, Q->h, H, 0);
    for (int64_t i = 0; i < T * H; ++i) Q->h[i] += Q->x[i];
    rmsnorm_fwd(T, H, Q->h, W[OB_NORM2], sh->eps, Q->n2, Q->r2);
    mm_nt(T, I, H, Q->n2, H, W[OB_GATE], H, Q->g, I, 0);
    mm_nt(T, I, H, Q->n2, H, W[OB_UP], H, Q->u, I, 0);
    for (int64_t i = 0; i < T * I; ++i) Q->a[i] = silu_f(Q->g[i]) * Q->u[i];
    mm_nt(T, H, I, Q->a, I, W[OB_DOWN], I, Q->y, H, 0);
    for (int64_t i = 0; i < T * H; ++i) Q->y[i] += Q->h[i];
    memcpy(y + r * T * H, Q->y, sizeof(float) * (size_t)(T * H));
  }

  /* ---------------- backward ---------------- */
  /* per-rank partial weight gradients (full size), reduce-scattered at the end */
  float** part = (float**)calloc((size_t)p * OB_COUNT, sizeof(float*));
  for (int r = 0; r < p; ++r)
    for (int t = 0; t < OB_COUNT; ++t) part[r * OB_COUNT + t] = zalloc(tensor_numel(sh, t));
  float** dh = (float**)calloc((size_t)p, sizeof(float*));
  float** dO_tok = (float**)calloc((size_t)p, sizeof(float*));
  float** dO_heads = (float**)calloc((size_t)p, sizeof(float*));
  float** dqkv_heads = (float**)calloc((size_t)p, sizeof(float*));
  float** dqkv_tok = (float**)calloc((size_t)p, sizeof(float*));

  for (int r = 0; r < p; ++r) {
    ob_rank* Q = &R[r];
    float** G = part + r * OB_COUNT;
    const float* dyr = dy + r * T * H;
    float* da = zalloc(T * I);
    float* dgu = zalloc(T * I);
    float* dn2 = zalloc(T * H);
    dh[r] = zalloc(T * H);
    memcpy(dh[r], dyr, sizeof(float) * (size_t)(T * H));
    /* down projection */
    mm_nn(T, I, H, dyr, H, W[OB_DOWN], I, da, I, 0);
    mm_tn(H, I, T, dyr, H, Q->a, I, G[OB_DOWN], I, 0);
    /* SwiGLU backward: dg into dgu, du into da (reuse) */
    for (int64_t i = 0; i < T * I; ++i) {
      const float gv = Q->g[i], sg = 1.f / (1.f + expf(-gv));
      const float dav = da[i];
      dgu[i] = dav * Q->u[i] * sg * (1.f + gv * (1.f - sg));
      da[i] = dav * gv * sg;
    }
    mm_nn(T, H, I, dgu, I, W[OB_GATE], H, dn2, H, 0);
    mm_nn(T, H, I, da, I, W[OB_UP], H, dn2, H, 1);
    mm_tn(I, H, T, dgu, I, Q->n2, H, G[OB_GATE], H, 0);
    mm_tn(I, H, T, da, I, Q->n2, H, G[OB_UP], H, 0);
    rmsnorm_bwd(T, H, Q->h, W[OB_NORM2], Q->r2, dn2, dh[r], G[OB_NORM2]);
    /* output projection */
    dO_tok[r] = zalloc(T * H);
    mm_nn(T, H, H, dh[r], H, W[OB_O], H, dO_tok[r], H, 0);
    mm_tn(H, H, T, dh[r], H, Q->o_tok, H, G[OB_O], H, 0);
    free(da); free(dgu); free(dn2);
  }
  for (int r = 0; r < p; ++r) {
    dO_heads[r] = zalloc(S * Hl);
    dqkv_heads[r] = zalloc(S * 3 * Hl);
    dqkv_tok[r] = zalloc(T * 3 * H);
  }
  a2a_tokens_to_heads(sh, p, dO_tok, H, dO_heads, Hl);
  for (int r = 0; r < p; ++r) {
    float* qh = R[r].qkv_heads;
    float* dq = dqkv_heads[r];
    attn_bwd(S, d, 0, Dl, qh, qh + Hl, qh + 2 * Hl, 3 * Hl, R[r].o_heads, dO_heads[r], Hl,
             R[r].lse, dq, dq + Hl, dq + 2 * Hl);
  }
  /* reverse all-to-all of dq|dk|dv: head-sharded -> token-sharded, per part */
  for (int part_i = 0; part_i < 3; ++part_i) {
    for (int dst = 0; dst < p; ++dst)
      for (int src = 0; src < p; ++src)
        for (int64_t t = 0; t < T; ++t)
          memcpy(dqkv_tok[dst] + t * 3 * H + part_i * H + src * Hl,
                 dqkv_heads[src] + (dst * T + t) * 3 * Hl + part_i * Hl, sizeof(float) * (size_t)Hl);
  }
  for (int r = 0; r < p; ++r) {
    ob_rank* Q = &R[r];
    float** G = part + r * OB_COUNT;
    rope_apply(T, Q->t0, sh, dqkv_tok[r], 3 * H, cos_t, sin_t, -1);
    float* dn1 = zalloc(T * H);
    mm_nn(T, H, 3 * H, dqkv_tok[r], 3 * H, W[OB_QKV], H, dn1, H, 0);
    mm_tn(3 * H, H, T, dqkv_tok[r], 3 * H, Q->n1, H, G[OB_QKV], H, 0);
    float* dxr = dx + r * T * H;
    memcpy(dxr, dh[r], sizeof(float) * (size_t)(T * H));
    rmsnorm_bwd(T, H, Q->x, W[OB_NORM1], Q->r1, dn1, dxr, G[OB_NORM1]);
    free(dn1);
  }
  /* reduce-scatter: rank r keeps sum over ranks of slice r (rank order) */
  for (int t = 0; t < OB_COUNT; ++t) {
    const int64_t n = tensor_numel(sh, t), per = n / p;
    for (int r = 0; r < p; ++r) {
      float* dst = grad[t] + r * per;
      for (int64_t i = 0; i < per; ++i) {
        float s = 0;
        for (int q = 0; q < p; ++q) s += part[q * OB_COUNT + t][r * per + i];
        dst[i] = s;
      }
    }
  }

  for (int r = 0; r < p; ++r) {
    for (int t = 0; t < OB_COUNT; ++t) free(part[r * OB_COUNT + t]);
    free(dh[r]); free(dO_tok[r]); free(dO_heads[r]); free(dqkv_heads[r]); free(dqkv_tok[r]);
    rank_free(&R[r]);
  }
  free(part); free(dh); free(dO_tok); free(dO_heads); free(dqkv_heads); free(dqkv_tok); free(R);
  for (int t = 0; t < OB_COUNT; ++t) free(W[t]);
  free(cos_t); free(sin_t);
  return 0;
}

void ob_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int ob_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* dot product with 16 partial sums (vectorisable without -ffast-math); d % 16 == 0 */
static inline float dot16(const float* a, const float* b, int64_t d) {
  float acc[16] = {0};
  for (int64_t k = 0; k < d; k += 16)
    for (int l = 0; l < 16; ++l) acc[l] += a[k + l] * b[k + l];
  float s = 0;
  for (int l = 0; l < 16; ++l) s += acc[l];
  return s;
}

/* ------------------------------------------------------------------------------------
 * Bounded sample of the block's work (bench.py's CPU baseline / reference arm; never a
 * parity path). The full fwd + bwd of n token rows at positions pos[] of an S-token sequence:
 * per-row norms, the QKV / O / gate / up / down GEMMs and all their gradients, RoPE, and the
 * causal attention of each row against its whole prefix, forward and backward (the row's
 * dK / dV contributions accumulate into dkv). kv [S, 2H] holds the rotated K | V of every
 * position (the caller prepares it outside the timed region; the sampled rows' own K, V are
 * written in). With n rows spread evenly over the sequence this is n/S of the block's FLOPs.
 * W: full weights (OB_* order); grad: full-size gradient accumulators.
 * ------------------------------------------------------------------------------------ */
int ob_block_sample(const ob_shape* sh, const float* const* W, const int64_t* pos, int64_t n,
                    const float* x, const float* dy, float* kv, float* dkv, float* y, float* dx,
                    float* const* grad) {
  const int64_t H = sh->H, D = sh->D, S = sh->S, I = sh->I, d = H / D;
  if (n < 1 || H % D || d % 16) return -1;
  for (int64_t i = 0; i < n; ++i)
    if (pos[i] < 0 || pos[i] >= S) return -1;
  const float scale = (float)(1.0 / sqrt((double)d));
  float* cos_t = zalloc(S * (d / 2));
  float* sin_t = zalloc(S * (d / 2));
  ob_rope_table(S, d, sh->rope_base, cos_t, sin_t);
  float *n1 = zalloc(n * H), *r1 = zalloc(n), *qkv = zalloc(n * 3 * H), *o = zalloc(n * H);
  float *lse = zalloc(n * D), *h = zalloc(n * H), *n2 = zalloc(n * H), *r2 = zalloc(n);
  float *g = zalloc(n * I), *u = zalloc(n * I), *a = zalloc(n * I);

  /* forward */
  rmsnorm_fwd(n, H, x, W[OB_NORM1], sh->eps, n1, r1);
  mm_nt(n, 3 * H, H, n1, H, W[OB_QKV], H, qkv, 3 * H, 0);
  for (int64_t i = 0; i < n; ++i) {
    rope_apply(1, pos[i], sh, qkv + i * 3 * H, 3 * H, cos_t, sin_t, +1);
    memcpy(kv + pos[i] * 2 * H, qkv + i * 3 * H + H, sizeof(float) * (size_t)(2 * H));
  }
  /* attention, head-parallel; keys in blocks of 64 shared by all rows (K / V read once per
   * block instead of once per row) */
  int64_t pmax = 0;
  for (int64_t i = 0; i < n; ++i) pmax = pos[i] > pmax ? pos[i] : pmax;
  const int64_t KB = 64;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t hh = 0; hh < D; ++hh) {
    float* sc = (float*)malloc(sizeof(float) * (size_t)(n * (pmax + 1)));
    const int64_t ld = pmax + 1;
    for (int64_t j0 = 0; j0 <= pmax; j0 += KB)
      for (int64_t i = 0; i < n; ++i) {
        const float* qr = qkv + i * 3 * H + hh * d;
        const int64_t j1 = j0 + KB - 1 < pos[i] ? j0 + KB - 1 : pos[i];
        for (int64_t j = j0; j <= j1; ++j) {
          const float* kr = kv + j * 2 * H + hh * d;
          sc[i * ld + j] = dot16(qr, kr, d) * scale;
        }
      }
    for (int64_t i = 0; i < n; ++i) {
      float* p = sc + i * ld;
      float mx = -INFINITY;
      for (int64_t j = 0; j <= pos[i]; ++j) mx = p[j] > mx ? p[j] : mx;
      double sum = 0;
      for (int64_t j = 0; j <= pos[i]; ++j) { p[j] = expf(p[j] - mx); sum += p[j]; }
      const float inv = (float)(1.0 / sum);
      for (int64_t j = 0; j <= pos[i]; ++j) p[j] *= inv;
      lse[i * D + hh] = mx + (float)log(sum);
      float* orow = o + i * H + hh * d;
      for (int64_t c = 0; c < d; ++c) orow[c] = 0;
    }
    for (int64_t j0 = 0; j0 <= pmax; j0 += KB)
      for (int64_t i = 0; i < n; ++i) {
        float* orow = o + i * H + hh * d;
        const int64_t j1 = j0 + KB - 1 < pos[i] ? j0 + KB - 1 : pos[i];
        for (int64_t j = j0; j <= j1; ++j) {
          const float w = sc[i * ld + j];
          const float* vr = kv + j * 2 * H + H + hh * d;
          for (int64_t c = 0; c < d; ++c) orow[c] += w * vr[c];
        }
      }
    free(sc);
  }
  mm_nt(n, H, H, o, H, W[OB_O], H, h, H, 0);
  for (int64_t i = 0; i < n * H; ++i) h[i] += x[i];
  rmsnorm_fwd(n, H, h, W[OB_NORM2], sh->eps, n2, r2);
  mm_nt(n, I, H, n2, H, W[OB_GATE], H, g, I, 0);
  mm_nt(n, I, H, n2, H, W[OB_UP], H, u, I, 0);
  for (int64_t i = 0; i < n * I; ++i) a[i] = silu_f(g[i]) * u[i];
  mm_nt(n, H, I, a, I, W[OB_DOWN], I, y, H, 0);
  for (int64_t i = 0; i < n * H; ++i) y[i] += h[i];

  /* backward */
  float *da = zalloc(n * I), *dgu = zalloc(n * I), *dn2 = zalloc(n * H), *dh = zalloc(n * H);
  float *dO = zalloc(n * H), *dqkv = zalloc(n * 3 * H), *dn1 = zalloc(n * H);
  memcpy(dh, dy, sizeof(float) * (size_t)(n * H));
  mm_nn(n, I, H, dy, H, W[OB_DOWN], I, da, I, 0);
  mm_tn(H, I, n, dy, H, a, I, grad[OB_DOWN], I, 1);
  for (int64_t i = 0; i < n * I; ++i) {
    const float gv = g[i], sg = 1.f / (1.f + expf(-gv)), dav = da[i];
    dgu[i] = dav * u[i] * sg * (1.f + gv * (1.f - sg));
    da[i] = dav * gv * sg;
  }
  mm_nn(n, H, I, dgu, I, W[OB_GATE], H, dn2, H, 0);
  mm_nn(n, H, I, da, I, W[OB_UP], H, dn2, H, 1);
  mm_tn(I, H, n, dgu, I, n2, H, grad[OB_GATE], H, 1);
  mm_tn(I, H, n, da, I, n2, H, grad[OB_UP], H, 1);
  rmsnorm_bwd(n, H, h, W[OB_NORM2], r2, dn2, dh, grad[OB_NORM2]);
  mm_nn(n, H, H, dh, H, W[OB_O], H, dO, H, 0);
  mm_tn(H, H, n, dh, H, o, H, grad[OB_O], H, 1);
  /* attention backward: head-parallel (every head's dK / dV columns have one writer), keys in
   * blocks shared by all rows as in the forward */
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t hh = 0; hh < D; ++hh) {
    const int64_t ld = pmax + 1;
    float* P = (float*)malloc(sizeof(float) * (size_t)(n * ld));
    float* dS = (float*)malloc(sizeof(float) * (size_t)(n * ld));
    float* Dt = (float*)malloc(sizeof(float) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) {
      const float* dor = dO + i * H + hh * d;
      const float* orow = o + i * H + hh * d;
      float acc = 0;
      for (int64_t c = 0; c < d; ++c) acc += dor[c] * orow[c];
      Dt[i] = acc;
    }
    for (int64_t j0 = 0; j0 <= pmax; j0 += KB)
      for (int64_t i = 0; i < n; ++i) {
        const float* qr = qkv + i * 3 * H + hh * d;
        const float* dor = dO + i * H + hh * d;
        const float Lse = lse[i * D + hh];
        const int64_t j1 = j0 + KB - 1 < pos[i] ? j0 + KB - 1 : pos[i];
        for (int64_t j = j0; j <= j1; ++j) {
          const float* kr = kv + j * 2 * H + hh * d;
          const float* vr = kr + H;
          const float sv = dot16(qr, kr, d), dp = dot16(dor, vr, d);
          const float pv = expf(sv * scale - Lse);
          P[i * ld + j] = pv;
          dS[i * ld + j] = pv * (dp - Dt[i]) * scale;
        }
      }
    for (int64_t j0 = 0; j0 <= pmax; j0 += KB)
      for (int64_t i = 0; i < n; ++i) {
        const float* qr = qkv + i * 3 * H + hh * d;
        const float* dor = dO + i * H + hh * d;
        float* dqr = dqkv + i * 3 * H + hh * d;
        const int64_t j1 = j0 + KB - 1 < pos[i] ? j0 + KB - 1 : pos[i];
        for (int64_t j = j0; j <= j1; ++j) {
          const float* kr = kv + j * 2 * H + hh * d;
          float* dkr = dkv + j * 2 * H + hh * d;
          float* dvr = dkr + H;
          const float ds = dS[i * ld + j], pv = P[i * ld + j];
          for (int64_t c = 0; c < d; ++c) {
            dqr[c] += ds * kr[c];
            dkr[c] += ds * qr[c];
            dvr[c] += pv * dor[c];
          }
        }
      }
    free(P); free(dS); free(Dt);
  }
  for (int64_t i = 0; i < n; ++i) {
    memcpy(dqkv + i * 3 * H + H, dkv + pos[i] * 2 * H, sizeof(float) * (size_t)(2 * H));
    rope_apply(1, pos[i], sh, dqkv + i * 3 * H, 3 * H, cos_t, sin_t, -1);
  }
  mm_nn(n, H, 3 * H, dqkv, 3 * H, W[OB_QKV], H, dn1, H, 0);
  mm_tn(3 * H, H, n, dqkv, 3 * H, n1, H, grad[OB_QKV], H, 1);
  memcpy(dx, dh, sizeof(float) * (size_t)(n * H));
  rmsnorm_bwd(n, H, x, W[OB_NORM1], r1, dn1, dx, grad[OB_NORM1]);

  free(da); free(dgu); free(dn2); free(dh); free(dO); free(dqkv); free(dn1);
  free(n1); free(r1); free(qkv); free(o); free(lse); free(h); free(n2); free(r2);
  free(g); free(u); free(a); free(cos_t); free(sin_t);
  return 0;
}
