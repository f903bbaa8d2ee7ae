/* apl_oracle.c — CPU ORACLE (test infrastructure only).
 *
 * Plain-C restatement of the data semantics of the reference's layout
 * conversion steps, used ONLY by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg as the checker. Nothing in
 * the product (paper_2302_02599_b200/) links, loads or calls this file.
 *
 * What is restated (reference file:line):
 *   step semantics at spec level   proj/src/layout.cpp:178-219 and
 *                                  proj/tests/helpers.hpp:282-311 (apply_step):
 *     all-gather  pops the last axis a of dims[d]
 *     shard-slice appends an unused axis a to dims[d]
 *     all-to-all  moves the last axis a of dims[d] to the end of dims[d2]
 *   placement                      "assignment is row-major coordinate ->
 *                                  device" (proj/include/autoplan/cluster.hpp:56)
 *                                  + SURVEY.md Appendix A: block index of a dim
 *                                  = mixed radix over its axis list, first
 *                                  listed axis most significant.
 *   data semantics (Appendix A)    AG(d,a):  out(c) = concat_j in(c[a:=j]) along d
 *                                  SL(d,a):  out(c) = chunk c_a of n_a along d of in(c)
 *                                  A2A(d->d2,a): out(c) = concat_j (chunk c_a of n_a
 *                                  along d2 of in(c[a:=j])) along d
 *
 * Two independent evaluations are provided: oracle_local() slices a global
 * tensor directly by a spec, oracle_apply_step() executes one step as the
 * per-axis-group collective above. Pinning (tests/test_oracle.py): replaying
 * every reference path (oracle/_ref, and the committed tests/golden paths)
 * step by step must equal direct slicing by the target spec for every
 * device, which is the SURVEY's 0-mismatch consistency proof re-run here.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>

#define OR_MAX_DIMS 8
#define OR_MAX_MESH 8

typedef struct {
  int32_t rank;
  int32_t mesh_rank;
  int32_t naxes[OR_MAX_DIMS];
  int32_t axes[OR_MAX_DIMS][OR_MAX_MESH];
} or_spec; /* layout-compatible with apl_spec */

static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* Synthetic conversion payload: element i gets the low
 * elem_bytes of splitmix64(i ^ seed); fp32/bf16-sized elements have an
 * all-ones exponent cleared so no NaN/Inf appears. Compared bytewise. */
void oracle_fill(uint8_t* out, int64_t n, int elem_bytes, uint64_t seed) {
  for (int64_t i = 0; i < n; ++i) {
    uint64_t bits = splitmix64((uint64_t)i ^ seed);
    if (elem_bytes == 4 && ((bits >> 23) & 0xFFu) == 0xFFu) bits &= ~(uint64_t)0x40000000u;
    if (elem_bytes == 2 && ((bits >> 7) & 0xFFu) == 0xFFu) bits &= ~(uint64_t)0x4000u;
    memcpy(out + i * elem_bytes, &bits, (size_t)elem_bytes);
  }
}

static int64_t dim_split(const or_spec* s, int d, const int64_t* mesh) {
  int64_t p = 1;
  for (int i = 0; i < s->naxes[d]; ++i) p *= mesh[s->axes[d][i]];
  return p;
}

static void coord_of(int64_t dev, const int64_t* mesh, int mr, int64_t* c) {
  for (int i = mr - 1; i >= 0; --i) {
    c[i] = dev % mesh[i];
    dev /= mesh[i];
  }
}

static int64_t device_of(const int64_t* c, const int64_t* mesh, int mr) {
  int64_t d = 0;
  for (int i = 0; i < mr; ++i) d = d * mesh[i] + c[i];
  return d;
}


/* Minimal pthread parallel-for over [0, n) (no OpenMP runtime in this image). */
static int g_threads = 1;
typedef void (*or_body)(int64_t i, void* ctx);
typedef struct {
  or_body fn;
  void* ctx;
  int64_t n, tid, nthreads;
} or_job;
static void* or_worker(void* p) {
  or_job* j = (or_job*)p;
  for (int64_t i = j->tid; i < j->n; i += j->nthreads) j->fn(i, j->ctx);
  return NULL;
}
static void or_parallel_for(int64_t n, or_body fn, void* ctx) {
  int64_t t = g_threads < n ? g_threads : n;
  if (t <= 1) {
    for (int64_t i = 0; i < n; ++i) fn(i, ctx);
    return;
  }
  pthread_t th[64];
  or_job jobs[64];
  if (t > 64) t = 64;
  for (int64_t k = 0; k < t; ++k) {
    jobs[k] = (or_job){fn, ctx, n, k, t};
    pthread_create(&th[k], NULL, or_worker, &jobs[k]);
  }
  for (int64_t k = 0; k < t; ++k) pthread_join(th[k], NULL);
}

/* Local shard of `global` for `device` under `spec`, by direct slicing. */
void oracle_local(const uint8_t* global, const int64_t* shape, int rank, int eb,
                  const int64_t* mesh, int mr, const or_spec* spec, int64_t device,
                  uint8_t* out) {
  int64_t c[OR_MAX_MESH], lo[OR_MAX_DIMS], L[OR_MAX_DIMS], gstride[OR_MAX_DIMS];
  coord_of(device, mesh, mr, c);
  int64_t total = 1;
  for (int d = 0; d < rank; ++d) {
    int64_t s = 0;
    for (int i = 0; i < spec->naxes[d]; ++i) s = s * mesh[spec->axes[d][i]] + c[spec->axes[d][i]];
    L[d] = shape[d] / dim_split(spec, d, mesh);
    lo[d] = s * L[d];
    total *= L[d];
  }
  gstride[rank - 1] = 1;
  for (int d = rank - 2; d >= 0; --d) gstride[d] = gstride[d + 1] * shape[d + 1];
  /* walk rows of the local block (last dim contiguous) */
  const int64_t row = L[rank - 1];
  const int64_t rows = total / row;
  for (int64_t r = 0; r < rows; ++r) {
    int64_t rest = r, goff = lo[rank - 1];
    for (int d = rank - 2; d >= 0; --d) {
      goff += (lo[d] + rest % L[d]) * gstride[d];
      rest /= L[d];
    }
    memcpy(out + r * row * eb, global + goff * eb, (size_t)(row * eb));
  }
}

/* [P, L, Q] helpers on row-major arrays, dim d of local shape `ls`. */
static void pq_of(const int64_t* ls, int rank, int d, int64_t* P, int64_t* Q) {
  *P = 1;
  *Q = 1;
  for (int i = 0; i < d; ++i) *P *= ls[i];
  for (int i = d + 1; i < rank; ++i) *Q *= ls[i];
}

/* One reference step on P simulated devices: in[dev] (local shards under
 * `src`) -> out[dev] (local shards under the step result).
 * kind: 0 all-gather, 3 all-to-all, 4 shard-slice (CollectiveKind order). */
typedef struct {
  int kind, tdim, target, axis, rank, eb, mr;
  const int64_t* mesh;
  int64_t ls[OR_MAX_DIMS];
  const uint8_t* const* in;
  uint8_t* const* out;
} step_ctx;

static void step_device(int64_t dev, void* p) {
  const step_ctx* s = (const step_ctx*)p;
  const int64_t eb = s->eb, na = s->mesh[s->axis];
  int64_t c[OR_MAX_MESH];
  coord_of(dev, s->mesh, s->mr, c);
  if (s->kind == 0) { /* all-gather: concat the group's shards along tdim */
    int64_t P, Q;
    pq_of(s->ls, s->rank, s->tdim, &P, &Q);
    const int64_t L = s->ls[s->tdim];
    for (int64_t j = 0; j < na; ++j) {
      c[s->axis] = j;
      const uint8_t* part = s->in[device_of(c, s->mesh, s->mr)];
      for (int64_t q = 0; q < P; ++q)
        memcpy(s->out[dev] + ((q * na + j) * L) * Q * eb, part + q * L * Q * eb,
               (size_t)(L * Q * eb));
    }
  } else if (s->kind == 4) { /* shard-slice: keep chunk c_axis of na along tdim */
    int64_t P, Q;
    pq_of(s->ls, s->rank, s->tdim, &P, &Q);
    const int64_t L = s->ls[s->tdim], l = L / na;
    for (int64_t q = 0; q < P; ++q)
      memcpy(s->out[dev] + q * l * Q * eb, s->in[dev] + (q * L + c[s->axis] * l) * Q * eb,
             (size_t)(l * Q * eb));
  } else { /* all-to-all: chunk c_axis along target from each peer, concat along tdim */
    int64_t cs[OR_MAX_DIMS];
    memcpy(cs, s->ls, sizeof(int64_t) * (size_t)s->rank);
    cs[s->target] = s->ls[s->target] / na;
    int64_t Pt, Qt, Pd, Qd;
    pq_of(s->ls, s->rank, s->target, &Pt, &Qt);
    pq_of(cs, s->rank, s->tdim, &Pd, &Qd);
    const int64_t Lt = s->ls[s->target], lt = cs[s->target], Ld = cs[s->tdim];
    int64_t chunk_elems = 1;
    for (int d = 0; d < s->rank; ++d) chunk_elems *= cs[d];
    const int64_t mine = c[s->axis];
    uint8_t* chunk = (uint8_t*)malloc((size_t)(chunk_elems * eb));
    for (int64_t j = 0; j < na; ++j) {
      c[s->axis] = j;
      const uint8_t* peer = s->in[device_of(c, s->mesh, s->mr)];
      for (int64_t q = 0; q < Pt; ++q)
        memcpy(chunk + q * lt * Qt * eb, peer + (q * Lt + mine * lt) * Qt * eb,
               (size_t)(lt * Qt * eb));
      for (int64_t q = 0; q < Pd; ++q)
        memcpy(s->out[dev] + ((q * na + j) * Ld) * Qd * eb, chunk + q * Ld * Qd * eb,
               (size_t)(Ld * Qd * eb));
    }
    free(chunk);
  }
}

int oracle_apply_step(int kind, int tdim, int target, int axis, const int64_t* shape, int rank,
                      int eb, const int64_t* mesh, int mr, const or_spec* src,
                      const uint8_t* const* in, uint8_t* const* out) {
  if (kind != 0 && kind != 3 && kind != 4) return 1;
  step_ctx s;
  s.kind = kind;
  s.tdim = tdim;
  s.target = target;
  s.axis = axis;
  s.rank = rank;
  s.eb = eb;
  s.mr = mr;
  s.mesh = mesh;
  s.in = in;
  s.out = out;
  int64_t ndev = 1;
  for (int i = 0; i < mr; ++i) ndev *= mesh[i];
  for (int d = 0; d < rank; ++d) s.ls[d] = shape[d] / dim_split(src, d, mesh);
  or_parallel_for(ndev, step_device, &s);
  return 0;
}

int oracle_num_threads(void) { return g_threads; }

void oracle_set_threads(int n) { g_threads = n > 0 ? (n > 64 ? 64 : n) : 1; }

/* Sum of group partials in member order with fp32 accumulation for the
 * partial-sum all-reduce check (dtype 0 f32, 1 bf16). */
static float bf16_to_f(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static uint16_t f_to_bf16(float f) { /* round to nearest even */
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return (uint16_t)(u >> 16);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
void oracle_group_sum(const void* const* parts, int nparts, int64_t count, int dtype,
                      void* out) {
  for (int64_t i = 0; i < count; ++i) {
    float acc = 0.f;
    for (int j = 0; j < nparts; ++j)
      acc += dtype == 0 ? ((const float*)parts[j])[i] : bf16_to_f(((const uint16_t*)parts[j])[i]);
    if (dtype == 0) ((float*)out)[i] = acc;
    else ((uint16_t*)out)[i] = f_to_bf16(acc);
  }
}
