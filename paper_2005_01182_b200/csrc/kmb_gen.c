/*
 * Seeded synthetic workloads for the five BASELINE.json configs (SURVEY.md
 * §8(d)).  The reference has no generator for them (its datasets.cpp has no
 * squared-Euclidean mode and no seeded uniform / GMM generators), so they are
 * defined here once, portably:
 *
 *   draw(stream, k, a) = splitmix64_mix(stream + (4k + a + 1) * GOLDEN)
 *
 * is a counter-based stream (element k, attempt a), so every element can be
 * generated independently (OpenMP) and the result does not depend on the
 * thread count.  Bounded integers use Lemire's multiply-shift with rejection
 * (unbiased); doubles are (x >> 11) * 2^-53; normals are Box-Muller in double
 * (cos branch).  Distances accumulate in double in dimension order with FP
 * contraction disabled (-ffp-contract=off), and are rounded with llround —
 * the same rounding the reference's build_instance uses (datasets.cpp:184-214).
 * Generated once on the host; the oracle and the GPU read the same int32
 * buffer.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline uint64_t stream_of(uint64_t seed, uint64_t tag) {
  return mix64(seed * GOLDEN + mix64(tag + 0x632BE59BD9B4E019ULL));
}

static inline uint64_t draw(uint64_t stream, uint64_t k, uint64_t a) {
  return mix64(stream + (4 * k + a + 1) * GOLDEN);
}

/* unbiased integer in [0, range) (Lemire 2019), range >= 1 */
static inline uint64_t bounded(uint64_t stream, uint64_t k, uint64_t range) {
  uint64_t a = 0;
  for (;;) {
    const uint64_t x = draw(stream, k, a++);
    const unsigned __int128 m = (unsigned __int128)x * range;
    const uint64_t lo = (uint64_t)m;
    if (lo >= range) return (uint64_t)(m >> 64);
    const uint64_t t = (0 - range) % range;
    if (lo >= t) return (uint64_t)(m >> 64);
  }
}

static inline double unit(uint64_t stream, uint64_t k, uint64_t a) {
  return (double)(draw(stream, k, a) >> 11) * 0x1.0p-53;
}

static inline double normal(uint64_t stream, uint64_t k) {
  const double u1 = unit(stream, k, 0), u2 = unit(stream, k, 1);
  return sqrt(-2.0 * log(1.0 - u1)) * cos(6.283185307179586476925 * u2);
}

/* Config 1 / 5 (and any uniform case): C[i][j] ~ U{lo..hi}, row-major. */
void kmb_gen_uniform(int32_t* out, int32_t n, int32_t lo, int32_t hi, uint64_t seed) {
  const uint64_t st = stream_of(seed, 1);
  const uint64_t range = (uint64_t)((int64_t)hi - lo + 1);
  const int64_t total = (int64_t)n * n;
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < total; ++k) out[k] = lo + (int32_t)bounded(st, (uint64_t)k, range);
}

/* Config 2: two sets of n points U[0,1)^2 (fp64);
 * C = llround(scale * squared Euclidean distance). */
void kmb_gen_geometric(int32_t* out, int32_t n, double scale, uint64_t seed) {
  double* a = malloc(sizeof(double) * 2 * (size_t)n);
  double* b = malloc(sizeof(double) * 2 * (size_t)n);
  const uint64_t sa = stream_of(seed, 2), sb = stream_of(seed, 3);
  for (int32_t p = 0; p < 2 * n; ++p) {
    a[p] = unit(sa, (uint64_t)p, 0);
    b[p] = unit(sb, (uint64_t)p, 0);
  }
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < n; ++i)
    for (int32_t j = 0; j < n; ++j) {
      const double dx = a[2 * i] - b[2 * j], dy = a[2 * i + 1] - b[2 * j + 1];
      const double d2 = dx * dx + dy * dy;
      out[(size_t)i * n + j] = (int32_t)llround(scale * d2);
    }
  free(a);
  free(b);
}

/* Config 3: instances first .. first+batch-1; instance t draws 2n vectors of
 * dimension dim, i.i.d. N(0,1) in fp32 from its own stream
 * stream_of(seed, 4<<32 | t) (so any shard of the batch can be generated alone);
 * C = llround(scale * Euclidean distance) with the distance in double. */
void kmb_gen_embedding_batch(int32_t* out, int32_t first, int32_t batch, int32_t n,
                             int32_t dim, double scale, uint64_t seed) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int32_t t = 0; t < batch; ++t) {
    const uint64_t st = stream_of(seed, (4ULL << 32) | (uint64_t)(first + t));
    float* x = malloc(sizeof(float) * 2 * (size_t)n * dim);
    for (int64_t k = 0; k < 2 * (int64_t)n * dim; ++k) x[k] = (float)normal(st, (uint64_t)k);
    const float* A = x;
    const float* Bv = x + (size_t)n * dim;
    int32_t* c = out + (size_t)t * n * n;
    for (int32_t i = 0; i < n; ++i)
      for (int32_t j = 0; j < n; ++j) {
        double s = 0.0;
        const float* p = A + (size_t)i * dim;
        const float* q = Bv + (size_t)j * dim;
        for (int32_t d = 0; d < dim; ++d) {
          const double diff = (double)p[d] - (double)q[d];
          s += diff * diff;
        }
        c[(size_t)i * n + j] = (int32_t)llround(scale * sqrt(s));
      }
    free(x);
  }
}

/* Config 4: two sets of n points in 3-D from a `comps`-component Gaussian
 * mixture (means U[0,box]^3, sigma per axis, uniform component choice, fp64);
 * C = llround(scale * squared Euclidean distance). */
void kmb_gen_gmm(int32_t* out, int32_t n, int32_t comps, double box, double sigma,
                 double scale, uint64_t seed) {
  double* mu = malloc(sizeof(double) * 3 * (size_t)comps);
  double* P[2];
  const uint64_t sm = stream_of(seed, 5);
  for (int32_t k = 0; k < 3 * comps; ++k) mu[k] = box * unit(sm, (uint64_t)k, 0);
  for (int s = 0; s < 2; ++s) {
    P[s] = malloc(sizeof(double) * 3 * (size_t)n);
    const uint64_t sc = stream_of(seed, 6 + 2 * (uint64_t)s);
    const uint64_t sz = stream_of(seed, 7 + 2 * (uint64_t)s);
    for (int32_t p = 0; p < n; ++p) {
      const int32_t comp = (int32_t)bounded(sc, (uint64_t)p, (uint64_t)comps);
      for (int d = 0; d < 3; ++d)
        P[s][3 * p + d] = mu[3 * comp + d] + sigma * normal(sz, (uint64_t)(3 * p + d));
    }
  }
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < n; ++i)
    for (int32_t j = 0; j < n; ++j) {
      double d2 = 0.0;
      for (int d = 0; d < 3; ++d) {
        const double diff = P[0][3 * i + d] - P[1][3 * j + d];
        d2 += diff * diff;
      }
      out[(size_t)i * n + j] = (int32_t)llround(scale * d2);
    }
  free(mu);
  free(P[0]);
  free(P[1]);
}

/* FNV-1a 64 over a byte buffer (fixture hashes of u, v, costs). */
uint64_t kmb_fnv1a64(const void* data, int64_t nbytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ULL;
  for (int64_t k = 0; k < nbytes; ++k) {
    h ^= p[k];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* ---- the point sets behind configs 2-4 (same streams as the cost generators
 * above), for GPU cost construction (csrc/kmb_costs.cu) ------------------ */

/* config 2: a, b = n x 2 doubles */
void kmb_gen_geometric_points(double* a, double* b, int32_t n, uint64_t seed) {
  const uint64_t sa = stream_of(seed, 2), sb = stream_of(seed, 3);
  for (int32_t p = 0; p < 2 * n; ++p) {
    a[p] = unit(sa, (uint64_t)p, 0);
    b[p] = unit(sb, (uint64_t)p, 0);
  }
}

/* config 4: a, b = n x 3 doubles */
void kmb_gen_gmm_points(double* a, double* b, int32_t n, int32_t comps, double box, double sigma,
                        uint64_t seed) {
  double* mu = malloc(sizeof(double) * 3 * (size_t)comps);
  const uint64_t sm = stream_of(seed, 5);
  for (int32_t k = 0; k < 3 * comps; ++k) mu[k] = box * unit(sm, (uint64_t)k, 0);
  for (int s = 0; s < 2; ++s) {
    double* P = s == 0 ? a : b;
    const uint64_t sc = stream_of(seed, 6 + 2 * (uint64_t)s);
    const uint64_t sz = stream_of(seed, 7 + 2 * (uint64_t)s);
    for (int32_t p = 0; p < n; ++p) {
      const int32_t comp = (int32_t)bounded(sc, (uint64_t)p, (uint64_t)comps);
      for (int d = 0; d < 3; ++d)
        P[3 * p + d] = mu[3 * comp + d] + sigma * normal(sz, (uint64_t)(3 * p + d));
    }
  }
  free(mu);
}

/* config 3: instances first..first+batch-1; a, b = batch x n x dim floats */
void kmb_gen_embedding_vectors(float* a, float* b, int32_t first, int32_t batch, int32_t n,
                               int32_t dim, uint64_t seed) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int32_t t = 0; t < batch; ++t) {
    const uint64_t st = stream_of(seed, (4ULL << 32) | (uint64_t)(first + t));
    const int64_t nd = (int64_t)n * dim;
    for (int64_t k = 0; k < nd; ++k) a[(size_t)t * nd + k] = (float)normal(st, (uint64_t)k);
    for (int64_t k = 0; k < nd; ++k) b[(size_t)t * nd + k] = (float)normal(st, (uint64_t)(nd + k));
  }
}
