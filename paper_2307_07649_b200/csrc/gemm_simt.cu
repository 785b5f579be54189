// Grouped fp32 SIMT GEMM (see gemm_simt.cuh).
#include "gemm_simt.cuh"

namespace tgb {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

struct GroupParams {
  GemmProblem p[kMaxGroup];
  int tiles_m[kMaxGroup], tiles_n[kMaxGroup];
  int count;
};

__device__ __forceinline__ int seg_of(const Operand& o, int k) {
  // Segment lookup along K (<= 4 segments).
  int s = 0;
#pragma unroll
  for (int x = 1; x < 4; ++x)
    if (x < o.nseg && k >= o.kb[x]) s = x;
  return s;
}

// A(m, k) = seg.p[m * rs + (k - kb) * cs]
__device__ __forceinline__ float a_at(const Operand& o, int64_t m, int k) {
  const int s = seg_of(o, k);
  const Seg& sg = o.seg[s];
  return sg.p[m * sg.rs + static_cast<int64_t>(k - o.kb[s]) * sg.cs];
}

// B(k, n) = seg.p[(k - kb) * rs + n * cs]
__device__ __forceinline__ float b_at(const Operand& o, int k, int64_t n) {
  const int s = seg_of(o, k);
  const Seg& sg = o.seg[s];
  return sg.p[static_cast<int64_t>(k - o.kb[s]) * sg.rs + n * sg.cs];
}

// A tile [BM x BK] -> As[k][m];  B tile [BK x BN] -> Bs[k][n].
__device__ __forceinline__ void load_a(const Operand& o, int m0, int k0, int M, int K, float (*As)[BM + 4],
                                       float* reg) {
  // Choose the mapping along the unit-stride direction of the first segment.
  const bool k_fast = o.seg[0].cs == 1;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = threadIdx.x + i * NT;
    int mm, kk;
    if (k_fast) {
      mm = idx / BK;
      kk = idx % BK;
    } else {
      kk = idx / BM;
      mm = idx % BM;
    }
    const int m = m0 + mm, k = k0 + kk;
    reg[i] = (m < M && k < K) ? a_at(o, m, k) : 0.0f;
  }
  (void)As;
}

__device__ __forceinline__ void store_a(const Operand& o, float (*As)[BM + 4], const float* reg) {
  const bool k_fast = o.seg[0].cs == 1;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = threadIdx.x + i * NT;
    int mm, kk;
    if (k_fast) {
      mm = idx / BK;
      kk = idx % BK;
    } else {
      kk = idx / BM;
      mm = idx % BM;
    }
    As[kk][mm] = reg[i];
  }
}

__device__ __forceinline__ void load_b(const Operand& o, int n0, int k0, int N, int K, float* reg) {
  const bool n_fast = o.seg[0].cs == 1;  // B(k, n): cs is the n-stride
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = threadIdx.x + i * NT;
    int nn, kk;
    if (n_fast) {
      kk = idx / BN;
      nn = idx % BN;
    } else {
      nn = idx / BK;
      kk = idx % BK;
    }
    const int n = n0 + nn, k = k0 + kk;
    reg[i] = (n < N && k < K) ? b_at(o, k, n) : 0.0f;
  }
}

__device__ __forceinline__ void store_b(const Operand& o, float (*Bs)[BN + 4], const float* reg) {
  const bool n_fast = o.seg[0].cs == 1;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = threadIdx.x + i * NT;
    int nn, kk;
    if (n_fast) {
      kk = idx / BN;
      nn = idx % BN;
    } else {
      nn = idx / BK;
      kk = idx % BK;
    }
    Bs[kk][nn] = reg[i];
  }
}

// B operand convention: B(k, n) = seg.p[k * rs + n * cs] (rows of B are k).
__global__ void __launch_bounds__(NT) gemm_group_kernel(const __grid_constant__ GroupParams gp) {
  const int pi = blockIdx.y;
  if (pi >= gp.count) return;
  const GemmProblem& P = gp.p[pi];
  const int tm = gp.tiles_m[pi], tn = gp.tiles_n[pi];
  const int tile = blockIdx.x;
  if (tile >= tm * tn * P.splits) return;
  const int split = tile / (tm * tn);
  const int t2 = tile % (tm * tn);
  const int m0 = (t2 / tn) * BM, n0 = (t2 % tn) * BN;
  const int M = P.M_dev ? min(P.M, *P.M_dev) : P.M;
  if (m0 >= M && P.splits == 1) return;
  const int N = P.N;
  const int Kcap = P.K;
  const int K = P.K_dev ? min(Kcap, *P.K_dev) : Kcap;
  // split-K range over the capacity (fixed partition => deterministic)
  const int kper = ((Kcap + P.splits - 1) / P.splits + BK - 1) / BK * BK;
  const int kbeg = split * kper;
  const int kend = min(K, kbeg + kper);

  __shared__ float As[2][BK][BM + 4];
  __shared__ float Bs[2][BK][BN + 4];

  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

  float ra[4], rb[4];
  int buf = 0;
  if (kbeg < kend && m0 < M) {
    load_a(P.a, m0, kbeg, M, kend, As[0], ra);
    load_b(P.b, n0, kbeg, N, kend, rb);
    store_a(P.a, As[0], ra);
    store_b(P.b, Bs[0], rb);
    __syncthreads();
    for (int k0 = kbeg; k0 < kend; k0 += BK) {
      const bool more = k0 + BK < kend;
      if (more) {
        load_a(P.a, m0, k0 + BK, M, kend, As[buf ^ 1], ra);
        load_b(P.b, n0, k0 + BK, N, kend, rb);
      }
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[buf][kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[buf][kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      if (more) {
        store_a(P.a, As[buf ^ 1], ra);
        store_b(P.b, Bs[buf ^ 1], rb);
      }
      __syncthreads();
      buf ^= 1;
    }
  }

  if (P.splits > 1) {
    float* ws = P.ws + static_cast<int64_t>(split) * P.M * P.N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + ty * 4 + i;
      if (m >= P.M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = n0 + tx * 4 + j;
        if (n < N) ws[static_cast<int64_t>(m) * N + n] = (m < M) ? acc[i][j] : 0.0f;
      }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float* c = P.C + static_cast<int64_t>(m) * P.ldc + n;
      float v = P.alpha * acc[i][j];
      if (P.beta != 0.0f) v += P.beta * *c;
      if (P.bias) v += P.bias[n];
      *c = v;
    }
  }
}

// In-order reduction of split-K partials into C.
__global__ void splitk_reduce_kernel(const __grid_constant__ GroupParams gp) {
  const int pi = blockIdx.y;
  const GemmProblem& P = gp.p[pi];
  if (P.splits <= 1) return;
  const int64_t total = static_cast<int64_t>(P.M) * P.N;
  for (int64_t x = blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float s = 0.0f;
    for (int sp = 0; sp < P.splits; ++sp) s += P.ws[sp * total + x];
    const int64_t m = x / P.N, n = x % P.N;
    float* c = P.C + m * P.ldc + n;
    float v = P.alpha * s;
    if (P.beta != 0.0f) v += P.beta * *c;
    if (P.bias) v += P.bias[n];
    *c = v;
  }
}

}  // namespace

namespace {
int g_impl = kGemmTma;
}

void set_gemm_impl(int impl) { g_impl = impl; }
int gemm_impl() { return g_impl; }

void splitk_reduce_launch(const GemmGroup& g, cudaStream_t s) {
  GroupParams gp{};
  gp.count = g.count;
  for (int i = 0; i < g.count; ++i) gp.p[i] = g.p[i];
  splitk_reduce_kernel<<<dim3(64, g.count), 256, 0, s>>>(gp);
  TGB_CUDA(cudaGetLastError());
}

void gemm_group_launch_tc(const GemmGroup& g, cudaStream_t s);

void gemm_group_launch(const GemmGroup& g, cudaStream_t s) {
  if (g_impl == kGemmGather) {
    gemm_group_launch_tc(g, s);
    return;
  }
  gemm_group_launch_simt(g, s);
}

void gemm_group_launch_simt(const GemmGroup& g, cudaStream_t s) {
  if (g.count == 0) return;
  GroupParams gp{};
  gp.count = g.count;
  int max_tiles = 0;
  bool any_split = false;
  for (int i = 0; i < g.count; ++i) {
    gp.p[i] = g.p[i];
    gp.tiles_m[i] = static_cast<int>(ceil_div(g.p[i].M, BM));
    gp.tiles_n[i] = static_cast<int>(ceil_div(g.p[i].N, BN));
    const int t = gp.tiles_m[i] * gp.tiles_n[i] * g.p[i].splits;
    max_tiles = t > max_tiles ? t : max_tiles;
    any_split |= g.p[i].splits > 1;
  }
  if (max_tiles == 0) return;
  gemm_group_kernel<<<dim3(max_tiles, g.count), NT, 0, s>>>(gp);
  TGB_CUDA(cudaGetLastError());
  if (any_split) splitk_reduce_launch(g, s);
}

}  // namespace tgb
