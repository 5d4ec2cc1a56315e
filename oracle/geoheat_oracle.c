/* TEST INFRASTRUCTURE ONLY — the CPU parity oracle, never the product.
 *
 * Plain-C restatement of the reference solver loop (arXiv 1812.06060 as
 * implemented by /root/reference/proj/include/geoheat). Each function cites
 * the reference file:line it follows and keeps the reference's evaluation
 * order operation by operation, so with FMA contraction off it reproduces the
 * reference bit for bit. It is pinned against the reference itself
 * (oracle/_ref/libgeoheat_ref.so, built by build_ref.sh) and against the
 * committed fixtures in tests/golden/ — see tests/test_oracle.py.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs load
 * it. Build: oracle/build_ref.sh (gcc -O2 -fopenmp -ffp-contract=off).
 */
#include "geoheat_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- vec3 ops
 * Eigen::Vector3d semantics as fixed in oracle/eigen_shim/Eigen/Core. */
typedef struct {
  double x, y, z;
} v3;
static inline v3 v3_make(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static inline v3 v3_sub(v3 a, v3 b) { return v3_make(a.x - b.x, a.y - b.y, a.z - b.z); }
static inline v3 v3_add(v3 a, v3 b) { return v3_make(a.x + b.x, a.y + b.y, a.z + b.z); }
static inline v3 v3_scale(double s, v3 a) { return v3_make(s * a.x, s * a.y, s * a.z); }
static inline v3 v3_div(v3 a, double s) { return v3_make(a.x / s, a.y / s, a.z / s); }
static inline double v3_dot(v3 a, v3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
static inline double v3_sqnorm(v3 a) { return v3_dot(a, a); }
static inline double v3_norm(v3 a) { return sqrt(v3_sqnorm(a)); }
static inline v3 v3_cross(v3 a, v3 b) {
  return v3_make(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static inline v3 v3_normalized(v3 a) {
  double n2 = v3_sqnorm(a);
  return n2 > 0.0 ? v3_div(a, sqrt(n2)) : a;
}
static inline v3 v3_load(const double* p, int64_t i) { return v3_make(p[3 * i], p[3 * i + 1], p[3 * i + 2]); }
static inline void v3_store(double* p, int64_t i, v3 a) { p[3 * i] = a.x; p[3 * i + 1] = a.y; p[3 * i + 2] = a.z; }

static int g_threads = 0; /* parallel.hpp:16-32 thread budget; 0 = hardware */
void gho_set_threads(int32_t threads) { g_threads = threads < 0 ? 0 : threads; }
static int thread_count(void) {
#ifdef _OPENMP
  return g_threads > 0 ? g_threads : omp_get_num_procs();
#else
  return 1;
#endif
}

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* ---------------------------------------------------------------- TriMesh */
struct gho_mesh {
  int32_t nv, nf, ne, ni;
  double* positions;       /* 3V */
  int32_t* faces;          /* 3F */
  int32_t* halfedge_twin;  /* 3F */
  int32_t* halfedge_edge;  /* 3F */
  int32_t* edge_vertices;  /* 2E */
  int32_t* edge_halfedges; /* 2E */
  int32_t* interior_edges; /* Eint */
  int32_t* interior_edge_index; /* E */
  uint8_t* vertex_on_boundary;  /* V */
  double* face_area;       /* F */
  double* face_normal;     /* 3F */
  double* vertex_area;     /* V */
  double* halfedge_cot;    /* 3F */
  double* edge_weight;     /* E */
  double* vertex_weight_sum; /* V */
  int32_t *vv_offset, *vv_index, *vv_edge;
  double* vv_weight;
  int32_t *vc_offset, *vc_corner;
};

void gho_mesh_free(gho_mesh* m) {
  if (!m) return;
  free(m->positions); free(m->faces); free(m->halfedge_twin); free(m->halfedge_edge);
  free(m->edge_vertices); free(m->edge_halfedges); free(m->interior_edges); free(m->interior_edge_index);
  free(m->vertex_on_boundary); free(m->face_area); free(m->face_normal); free(m->vertex_area);
  free(m->halfedge_cot); free(m->edge_weight); free(m->vertex_weight_sum); free(m->vv_offset);
  free(m->vv_index); free(m->vv_edge); free(m->vv_weight); free(m->vc_offset); free(m->vc_corner);
  free(m);
}

void gho_mesh_counts(const gho_mesh* m, int32_t counts[4]) {
  counts[0] = m->nv; counts[1] = m->nf; counts[2] = m->ne; counts[3] = m->ni;
}

const void* gho_mesh_array(const gho_mesh* m, int32_t which, int64_t* count) {
  const int64_t V = m->nv, F = m->nf, E = m->ne;
  switch (which) {
    case GHO_POSITIONS: *count = 3 * V; return m->positions;
    case GHO_FACES: *count = 3 * F; return m->faces;
    case GHO_HALFEDGE_TWIN: *count = 3 * F; return m->halfedge_twin;
    case GHO_HALFEDGE_EDGE: *count = 3 * F; return m->halfedge_edge;
    case GHO_EDGE_VERTICES: *count = 2 * E; return m->edge_vertices;
    case GHO_EDGE_HALFEDGES: *count = 2 * E; return m->edge_halfedges;
    case GHO_INTERIOR_EDGES: *count = m->ni; return m->interior_edges;
    case GHO_INTERIOR_EDGE_INDEX: *count = E; return m->interior_edge_index;
    case GHO_VERTEX_ON_BOUNDARY: *count = V; return m->vertex_on_boundary;
    case GHO_FACE_AREA: *count = F; return m->face_area;
    case GHO_FACE_NORMAL: *count = 3 * F; return m->face_normal;
    case GHO_VERTEX_AREA: *count = V; return m->vertex_area;
    case GHO_HALFEDGE_COT: *count = 3 * F; return m->halfedge_cot;
    case GHO_EDGE_WEIGHT: *count = E; return m->edge_weight;
    case GHO_VERTEX_WEIGHT_SUM: *count = V; return m->vertex_weight_sum;
    case GHO_VV_OFFSET: *count = V + 1; return m->vv_offset;
    case GHO_VV_INDEX: *count = 2 * E; return m->vv_index;
    case GHO_VV_EDGE: *count = 2 * E; return m->vv_edge;
    case GHO_VV_WEIGHT: *count = 2 * E; return m->vv_weight;
    case GHO_VC_OFFSET: *count = V + 1; return m->vc_offset;
    case GHO_VC_CORNER: *count = 3 * F; return m->vc_corner;
    default: *count = 0; return NULL;
  }
}

static inline int32_t he_tail(const gho_mesh* m, int64_t h) { return m->faces[h]; } /* faces[h/3][h%3] */
static inline int32_t he_head(const gho_mesh* m, int64_t h) {
  int64_t f = h / 3;
  return m->faces[3 * f + (h % 3 + 1) % 3];
}

/* cot_at (mesh.hpp:102-106) */
static double cot_at(v3 apex, v3 p, v3 q) {
  v3 u = v3_sub(p, apex), v = v3_sub(q, apex);
  return v3_dot(u, v) / v3_norm(v3_cross(u, v));
}

typedef struct {
  int32_t vmin, vmax, h;
} he_key;
static int cmp_he_key(const void* a, const void* b) {
  const he_key* x = (const he_key*)a;
  const he_key* y = (const he_key*)b;
  if (x->vmin != y->vmin) return x->vmin < y->vmin ? -1 : 1;
  if (x->vmax != y->vmax) return x->vmax < y->vmax ? -1 : 1;
  return (x->h > y->h) - (x->h < y->h);
}
typedef struct {
  int32_t nb, e;
} row_pair;
static int cmp_row_pair(const void* a, const void* b) {
  const row_pair* x = (const row_pair*)a;
  const row_pair* y = (const row_pair*)b;
  if (x->nb != y->nb) return x->nb < y->nb ? -1 : 1;
  return (x->e > y->e) - (x->e < y->e);
}

/* build_mesh (mesh.hpp:113-286) */
int gho_build_mesh(const double* positions, int32_t nv, const int32_t* faces, int32_t nf, gho_mesh** out,
                   char* err, int32_t errlen) {
  gho_mesh* m = (gho_mesh*)calloc(1, sizeof(gho_mesh));
  const int64_t V = nv, F = nf;
  m->nv = nv;
  m->nf = nf;
  m->positions = (double*)malloc(sizeof(double) * (3 * V + 1));
  m->faces = (int32_t*)malloc(sizeof(int32_t) * (3 * F + 1));
  memcpy(m->positions, positions, sizeof(double) * 3 * V);
  memcpy(m->faces, faces, sizeof(int32_t) * 3 * F);
#define FAIL(...)                                            \
  do {                                                       \
    if (err && errlen > 0) snprintf(err, errlen, __VA_ARGS__); \
    gho_mesh_free(m);                                        \
    return 1;                                                \
  } while (0)

  /* bbox -> degenerate threshold (120-126) */
  v3 lo = v3_make(INFINITY, INFINITY, INFINITY), hi = v3_make(-INFINITY, -INFINITY, -INFINITY);
  for (int64_t i = 0; i < V; ++i) {
    v3 p = v3_load(m->positions, i);
    /* std::min(a,b) = (b < a) ? b : a ; std::max(a,b) = (a < b) ? b : a */
    lo.x = p.x < lo.x ? p.x : lo.x; lo.y = p.y < lo.y ? p.y : lo.y; lo.z = p.z < lo.z ? p.z : lo.z;
    hi.x = hi.x < p.x ? p.x : hi.x; hi.y = hi.y < p.y ? p.y : hi.y; hi.z = hi.z < p.z ? p.z : hi.z;
  }
  const double bbox_diag2 = V > 0 ? v3_sqnorm(v3_sub(hi, lo)) : 0.0;
  const double degenerate_area = 1e-14 * bbox_diag2;

  /* face geometry and checks (128-145) */
  m->face_area = (double*)malloc(sizeof(double) * (F + 1));
  m->face_normal = (double*)malloc(sizeof(double) * (3 * F + 1));
  for (int64_t f = 0; f < F; ++f) {
    const int32_t* t = m->faces + 3 * f;
    for (int k = 0; k < 3; ++k)
      if (t[k] < 0 || t[k] >= nv) FAIL("face %lld: vertex index out of range", (long long)f);
    if (t[0] == t[1] || t[1] == t[2] || t[0] == t[2])
      FAIL("face %lld: repeated vertex (degenerate face)", (long long)f);
    v3 p0 = v3_load(m->positions, t[0]), p1 = v3_load(m->positions, t[1]), p2 = v3_load(m->positions, t[2]);
    v3 n = v3_cross(v3_sub(p1, p0), v3_sub(p2, p0));
    double area = 0.5 * v3_norm(n);
    if (!(area > degenerate_area)) FAIL("face %lld: degenerate (area %f)", (long long)f, area);
    m->face_area[f] = area;
    v3_store(m->face_normal, f, v3_div(n, 2.0 * area));
  }

  /* edges from sorted halfedge keys (147-192) */
  he_key* keys = (he_key*)malloc(sizeof(he_key) * (3 * F + 1));
  for (int64_t h = 0; h < 3 * F; ++h) {
    int32_t a = he_tail(m, h), b = he_head(m, h);
    keys[h].vmin = a < b ? a : b;
    keys[h].vmax = a < b ? b : a;
    keys[h].h = (int32_t)h;
  }
  qsort(keys, (size_t)(3 * F), sizeof(he_key), cmp_he_key);
  m->halfedge_twin = (int32_t*)malloc(sizeof(int32_t) * (3 * F + 1));
  m->halfedge_edge = (int32_t*)malloc(sizeof(int32_t) * (3 * F + 1));
  for (int64_t h = 0; h < 3 * F; ++h) m->halfedge_twin[h] = m->halfedge_edge[h] = -1;
  int64_t ecap = 3 * F + 1;
  m->edge_vertices = (int32_t*)malloc(sizeof(int32_t) * 2 * ecap);
  m->edge_halfedges = (int32_t*)malloc(sizeof(int32_t) * 2 * ecap);
  int64_t ne = 0;
  for (int64_t i = 0; i < 3 * F;) {
    int64_t j = i;
    while (j < 3 * F && keys[j].vmin == keys[i].vmin && keys[j].vmax == keys[i].vmax) ++j;
    int64_t incident = j - i;
    if (incident > 2) {
      int32_t a = keys[i].vmin, b = keys[i].vmax;
      free(keys);
      FAIL("non-manifold edge (%d,%d): %lld incident faces", a, b, (long long)incident);
    }
    int64_t e = ne++;
    m->edge_vertices[2 * e] = keys[i].vmin;
    m->edge_vertices[2 * e + 1] = keys[i].vmax;
    int32_t halves[2] = {-1, -1};
    for (int64_t k = i; k < j; ++k) {
      int32_t h = keys[k].h;
      m->halfedge_edge[h] = (int32_t)e;
      int side = he_tail(m, h) == keys[i].vmin ? 0 : 1;
      if (halves[side] >= 0) {
        int32_t a = keys[i].vmin, b = keys[i].vmax;
        free(keys);
        FAIL("inconsistent winding across edge (%d,%d)", a, b);
      }
      halves[side] = h;
    }
    if (incident == 2) {
      m->halfedge_twin[halves[0]] = halves[1];
      m->halfedge_twin[halves[1]] = halves[0];
    }
    m->edge_halfedges[2 * e] = halves[0];
    m->edge_halfedges[2 * e + 1] = halves[1];
    i = j;
  }
  free(keys);
  m->ne = (int32_t)ne;
  const int64_t E = ne;

  /* interior edges (194-201) */
  m->interior_edge_index = (int32_t*)malloc(sizeof(int32_t) * (E + 1));
  m->interior_edges = (int32_t*)malloc(sizeof(int32_t) * (E + 1));
  int64_t ni = 0;
  for (int64_t e = 0; e < E; ++e) {
    m->interior_edge_index[e] = -1;
    if (m->edge_halfedges[2 * e] >= 0 && m->edge_halfedges[2 * e + 1] >= 0) {
      m->interior_edge_index[e] = (int32_t)ni;
      m->interior_edges[ni++] = (int32_t)e;
    }
  }
  m->ni = (int32_t)ni;

  /* cotangents (203-213), edge weights theta (214-220) */
  m->halfedge_cot = (double*)malloc(sizeof(double) * (3 * F + 1));
  for (int64_t f = 0; f < F; ++f) {
    const int32_t* t = m->faces + 3 * f;
    v3 p0 = v3_load(m->positions, t[0]), p1 = v3_load(m->positions, t[1]), p2 = v3_load(m->positions, t[2]);
    m->halfedge_cot[3 * f + 0] = cot_at(p2, p0, p1);
    m->halfedge_cot[3 * f + 1] = cot_at(p0, p1, p2);
    m->halfedge_cot[3 * f + 2] = cot_at(p1, p2, p0);
  }
  m->edge_weight = (double*)malloc(sizeof(double) * (E + 1));
  for (int64_t e = 0; e < E; ++e) {
    double sum = 0.0;
    for (int s = 0; s < 2; ++s) {
      int32_t h = m->edge_halfedges[2 * e + s];
      if (h >= 0) sum += m->halfedge_cot[h];
    }
    m->edge_weight[e] = 0.5 * sum;
  }

  /* vertex areas in ascending face order (222-224) */
  m->vertex_area = (double*)calloc((size_t)V + 1, sizeof(double));
  for (int64_t f = 0; f < F; ++f)
    for (int k = 0; k < 3; ++k) m->vertex_area[m->faces[3 * f + k]] += m->face_area[f] / 3.0;

  /* boundary flags (226-232) */
  m->vertex_on_boundary = (uint8_t*)calloc((size_t)V + 1, 1);
  for (int64_t e = 0; e < E; ++e) {
    if (!(m->edge_halfedges[2 * e] >= 0 && m->edge_halfedges[2 * e + 1] >= 0)) {
      m->vertex_on_boundary[m->edge_vertices[2 * e]] = 1;
      m->vertex_on_boundary[m->edge_vertices[2 * e + 1]] = 1;
    }
  }

  /* CSR adjacency with rows sorted by neighbor (234-266) */
  m->vv_offset = (int32_t*)calloc((size_t)V + 1, sizeof(int32_t));
  for (int64_t e = 0; e < E; ++e) {
    m->vv_offset[m->edge_vertices[2 * e] + 1]++;
    m->vv_offset[m->edge_vertices[2 * e + 1] + 1]++;
  }
  for (int64_t v = 0; v < V; ++v) m->vv_offset[v + 1] += m->vv_offset[v];
  m->vv_index = (int32_t*)malloc(sizeof(int32_t) * (2 * E + 1));
  m->vv_edge = (int32_t*)malloc(sizeof(int32_t) * (2 * E + 1));
  m->vv_weight = (double*)malloc(sizeof(double) * (2 * E + 1));
  {
    int32_t* cursor = (int32_t*)malloc(sizeof(int32_t) * (V + 1));
    memcpy(cursor, m->vv_offset, sizeof(int32_t) * V);
    for (int64_t e = 0; e < E; ++e) {
      int32_t a = m->edge_vertices[2 * e], b = m->edge_vertices[2 * e + 1];
      m->vv_index[cursor[a]] = b;
      m->vv_edge[cursor[a]++] = (int32_t)e;
      m->vv_index[cursor[b]] = a;
      m->vv_edge[cursor[b]++] = (int32_t)e;
    }
    free(cursor);
    row_pair* row = (row_pair*)malloc(sizeof(row_pair) * 64);
    int64_t rowcap = 64;
    for (int64_t v = 0; v < V; ++v) {
      int32_t begin = m->vv_offset[v], end = m->vv_offset[v + 1];
      if (end - begin > rowcap) {
        rowcap = end - begin;
        row = (row_pair*)realloc(row, sizeof(row_pair) * rowcap);
      }
      for (int32_t i = begin; i < end; ++i) {
        row[i - begin].nb = m->vv_index[i];
        row[i - begin].e = m->vv_edge[i];
      }
      qsort(row, (size_t)(end - begin), sizeof(row_pair), cmp_row_pair);
      for (int32_t i = begin; i < end; ++i) {
        m->vv_index[i] = row[i - begin].nb;
        m->vv_edge[i] = row[i - begin].e;
        m->vv_weight[i] = m->edge_weight[row[i - begin].e];
      }
    }
    free(row);
  }
  /* row sums (267-270) */
  m->vertex_weight_sum = (double*)calloc((size_t)V + 1, sizeof(double));
  for (int64_t v = 0; v < V; ++v)
    for (int32_t i = m->vv_offset[v]; i < m->vv_offset[v + 1]; ++i) m->vertex_weight_sum[v] += m->vv_weight[i];

  /* vertex -> corner CSR in face order (272-283) */
  m->vc_offset = (int32_t*)calloc((size_t)V + 1, sizeof(int32_t));
  for (int64_t c = 0; c < 3 * F; ++c) m->vc_offset[m->faces[c] + 1]++;
  for (int64_t v = 0; v < V; ++v) m->vc_offset[v + 1] += m->vc_offset[v];
  m->vc_corner = (int32_t*)malloc(sizeof(int32_t) * (3 * F + 1));
  {
    int32_t* cursor = (int32_t*)malloc(sizeof(int32_t) * (V + 1));
    memcpy(cursor, m->vc_offset, sizeof(int32_t) * V);
    for (int64_t c = 0; c < 3 * F; ++c) m->vc_corner[cursor[m->faces[c]]++] = (int32_t)c;
    free(cursor);
  }
#undef FAIL
  *out = m;
  return 0;
}

/* edge_vector / edge_length (mesh.hpp:66-72) */
static inline v3 edge_vector(const gho_mesh* m, int64_t e) {
  return v3_sub(v3_load(m->positions, m->edge_vertices[2 * e + 1]), v3_load(m->positions, m->edge_vertices[2 * e]));
}

/* average_edge_length (mesh.hpp:289-293) */
double gho_average_edge_length(const gho_mesh* m) {
  double sum = 0.0;
  for (int64_t e = 0; e < m->ne; ++e) sum += v3_norm(edge_vector(m, e));
  return sum / (double)m->ne;
}

/* triangulation_quality (mesh.hpp:297-310) */
double gho_triangulation_quality(const gho_mesh* m) {
  double sum = 0.0;
  for (int64_t f = 0; f < m->nf; ++f) {
    const int32_t* t = m->faces + 3 * f;
    v3 p0 = v3_load(m->positions, t[0]), p1 = v3_load(m->positions, t[1]), p2 = v3_load(m->positions, t[2]);
    double a = v3_norm(v3_sub(p1, p2));
    double b = v3_norm(v3_sub(p2, p0));
    double c = v3_norm(v3_sub(p0, p1));
    double s = 0.5 * (a + b + c);
    double inradius = m->face_area[f] / s;
    double longest = a;
    if (longest < b) longest = b;
    if (longest < c) longest = c;
    sum += 2.0 * sqrt(3.0) * inradius / longest;
  }
  return sum / (double)m->nf;
}

/* edge_between (mesh.hpp:87-93): lower_bound in a's sorted row */
static int32_t edge_between(const gho_mesh* m, int32_t a, int32_t b) {
  int32_t lo = m->vv_offset[a], hi = m->vv_offset[a + 1];
  while (lo < hi) {
    int32_t mid = lo + (hi - lo) / 2;
    if (m->vv_index[mid] < b) lo = mid + 1;
    else hi = mid;
  }
  if (lo == m->vv_offset[a + 1] || m->vv_index[lo] != b) return -1;
  return m->vv_edge[lo];
}

/* face_gradient (mesh.hpp:314-327) */
void gho_face_gradient(const gho_mesh* m, const double* u, double* grad) {
  for (int64_t f = 0; f < m->nf; ++f) {
    const int32_t* t = m->faces + 3 * f;
    v3 n = v3_load(m->face_normal, f);
    v3 g = v3_make(0.0, 0.0, 0.0);
    for (int k = 0; k < 3; ++k) {
      v3 opp = v3_sub(v3_load(m->positions, t[(k + 2) % 3]), v3_load(m->positions, t[(k + 1) % 3]));
      g = v3_add(g, v3_scale(u[t[k]], v3_cross(n, opp)));
    }
    v3_store(grad, f, v3_div(g, 2.0 * m->face_area[f]));
  }
}

/* ---------------------------------------------------------------- BFS */
struct gho_levels {
  int32_t nv, nlev, unreachable;
  int32_t* level_of_vertex;
  int32_t* parent_of_vertex;
  int32_t* order;   /* concatenated rings */
  int32_t* offsets; /* nlev + 1 */
};

void gho_levels_free(gho_levels* l) {
  if (!l) return;
  free(l->level_of_vertex); free(l->parent_of_vertex); free(l->order); free(l->offsets); free(l);
}
void gho_levels_info(const gho_levels* l, int32_t info[2]) { info[0] = l->nlev; info[1] = l->unreachable; }
void gho_levels_get(const gho_levels* l, int32_t* lv, int32_t* par, int32_t* order, int32_t* offsets) {
  if (lv) memcpy(lv, l->level_of_vertex, sizeof(int32_t) * l->nv);
  if (par) memcpy(par, l->parent_of_vertex, sizeof(int32_t) * l->nv);
  if (order) memcpy(order, l->order, sizeof(int32_t) * l->offsets[l->nlev]);
  if (offsets) memcpy(offsets, l->offsets, sizeof(int32_t) * (l->nlev + 1));
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* bfs_levels (bfs.hpp:26-72) */
int gho_bfs(const gho_mesh* m, const int32_t* sources, int32_t ns, gho_levels** out, char* err, int32_t errlen) {
  const int64_t V = m->nv;
  if (ns <= 0) {
    if (err && errlen > 0) snprintf(err, errlen, "bfs_levels: empty source set");
    return 2;
  }
  for (int32_t i = 0; i < ns; ++i)
    if (sources[i] < 0 || sources[i] >= m->nv) {
      if (err && errlen > 0) snprintf(err, errlen, "bfs_levels: source index out of range");
      return 2;
    }
  gho_levels* l = (gho_levels*)calloc(1, sizeof(gho_levels));
  l->nv = m->nv;
  l->level_of_vertex = (int32_t*)malloc(sizeof(int32_t) * (V + 1));
  l->parent_of_vertex = (int32_t*)malloc(sizeof(int32_t) * (V + 1));
  for (int64_t v = 0; v < V; ++v) l->level_of_vertex[v] = l->parent_of_vertex[v] = -1;
  l->order = (int32_t*)malloc(sizeof(int32_t) * (V + 1));
  int64_t cap_off = 64;
  l->offsets = (int32_t*)malloc(sizeof(int32_t) * cap_off);

  /* D_0 = sorted unique sources (56-60) */
  int32_t* front = (int32_t*)malloc(sizeof(int32_t) * ns);
  memcpy(front, sources, sizeof(int32_t) * ns);
  qsort(front, ns, sizeof(int32_t), cmp_i32);
  int64_t n0 = 0;
  for (int32_t i = 0; i < ns; ++i)
    if (n0 == 0 || front[n0 - 1] != front[i]) front[n0++] = front[i];
  int64_t total = 0;
  l->offsets[0] = 0;
  for (int64_t i = 0; i < n0; ++i) {
    l->level_of_vertex[front[i]] = 0;
    l->order[total++] = front[i];
  }
  free(front);
  int32_t nlev = 1;
  l->offsets[1] = (int32_t)total;

  /* grow rings (61-86) */
  while (1) {
    const int32_t depth = nlev;
    const int64_t pb = l->offsets[nlev - 1], pe = l->offsets[nlev];
    int64_t nb = total;
    for (int64_t i = pb; i < pe; ++i) {
      int32_t v = l->order[i];
      for (int32_t a = m->vv_offset[v]; a < m->vv_offset[v + 1]; ++a) {
        int32_t w = m->vv_index[a];
        if (l->level_of_vertex[w] < 0) {
          l->level_of_vertex[w] = depth;
          l->order[total++] = w;
        }
      }
    }
    if (total == nb) break;
    qsort(l->order + nb, (size_t)(total - nb), sizeof(int32_t), cmp_i32);
    for (int64_t i = nb; i < total; ++i) {
      int32_t v = l->order[i];
      for (int32_t a = m->vv_offset[v]; a < m->vv_offset[v + 1]; ++a) {
        int32_t w = m->vv_index[a];
        if (l->level_of_vertex[w] == depth - 1) {
          l->parent_of_vertex[v] = w;
          break;
        }
      }
    }
    if (nlev + 2 > cap_off) {
      cap_off *= 2;
      l->offsets = (int32_t*)realloc(l->offsets, sizeof(int32_t) * cap_off);
    }
    ++nlev;
    l->offsets[nlev] = (int32_t)total;
  }
  l->nlev = nlev;
  l->unreachable = (int32_t)(V - total);
  *out = l;
  return 0;
}

/* ---------------------------------------------------------------- diffusion */

static void gs_sweep(const gho_mesh* m, const gho_levels* l, double t, const double* u0, double* u,
                     double* level_prev, int threads) {
  const int32_t* lov = l->level_of_vertex;
#pragma omp parallel num_threads(threads) if (threads > 1)
  for (int32_t li = 0; li < l->nlev; ++li) {
    const int32_t b = l->offsets[li], e = l->offsets[li + 1];
#pragma omp for schedule(static)
    for (int32_t i = b; i < e; ++i) level_prev[l->order[i]] = u[l->order[i]];
#pragma omp for schedule(static)
    for (int32_t i = b; i < e; ++i) {
      const int32_t j = l->order[i];
      double num = 0.0;
      for (int32_t a = m->vv_offset[j]; a < m->vv_offset[j + 1]; ++a) {
        const int32_t k = m->vv_index[a];
        const double value = lov[k] == li ? level_prev[k] : u[k];
        num += m->vv_weight[a] * value;
      }
      const double den = m->vertex_area[j] + t * m->vertex_weight_sum[j];
      u[j] = (u0[j] + t * num) / den;
    }
  }
}

/* gs_diffuse (diffusion.hpp:57-124): BFS-ordered Gauss-Seidel, Jacobi within
 * a level. With threads > 1 each level is split statically, as the reference
 * does under OpenMP; the result does not depend on the split. With tolerance
 * >= 0, E1 is evaluated after every sweep and the loop stops once E1 <= tol
 * (diffusion.hpp:110-117). */
static int diffuse(const gho_mesh* m, const gho_levels* l, double t, int32_t sweeps, double tolerance,
                   const double* initial, double* u, gho_report* report) {
  if (sweeps < 0 || !(t > 0.0)) return 2;
  double t0 = now_seconds();
  const int64_t V = m->nv;
  double* u0 = (double*)calloc((size_t)V + 1, sizeof(double));
  for (int64_t v = 0; v < V; ++v) u[v] = 0.0;
  for (int32_t i = l->offsets[0]; i < l->offsets[1]; ++i) {
    u0[l->order[i]] = 1.0;
    u[l->order[i]] = 1.0;
  }
  if (initial) memcpy(u, initial, sizeof(double) * V);
  double* level_prev = (double*)calloc((size_t)V + 1, sizeof(double));
  const int threads = thread_count();
  int32_t done = 0, converged = 0;
  for (int32_t sweep = 0; sweep < sweeps; ++sweep) {
    gs_sweep(m, l, t, u0, u, level_prev, threads);
    ++done;
    if (tolerance >= 0.0) {
      const double e1 = gho_diffusion_residual(m, u, t, l->order, l->offsets[1]);
      if (report && report->primal_history && sweep < report->history_capacity) report->primal_history[sweep] = e1;
      if (e1 <= tolerance) {
        converged = 1;
        break;
      }
    }
  }
  free(level_prev);
  free(u0);
  if (report) {
    report->iterations = done;
    report->converged = converged;
    report->wall_seconds = now_seconds() - t0;
  }
  return 0;
}

int gho_gs_diffuse(const gho_mesh* m, const gho_levels* l, double t, int32_t sweeps, const double* initial,
                   double* u, gho_report* report) {
  return diffuse(m, l, t, sweeps, -1.0, initial, u, report);
}

int gho_gs_diffuse_tol(const gho_mesh* m, const gho_levels* l, double t, int32_t sweeps, double tolerance,
                       const double* initial, double* u, gho_report* report) {
  return diffuse(m, l, t, sweeps, tolerance, initial, u, report);
}

/* diffusion_residual (diffusion.hpp:35-49) */
double gho_diffusion_residual(const gho_mesh* m, const double* u, double t, const int32_t* sources, int32_t ns) {
  const int64_t V = m->nv;
  double* u0 = (double*)calloc((size_t)V + 1, sizeof(double));
  for (int32_t i = 0; i < ns; ++i) u0[sources[i]] = 1.0;
  double sum = 0.0;
  for (int64_t j = 0; j < V; ++j) {
    double lap = 0.0;
    for (int32_t i = m->vv_offset[j]; i < m->vv_offset[j + 1]; ++i)
      lap += m->vv_weight[i] * (u[m->vv_index[i]] - u[j]);
    double r = m->vertex_area[j] * u[j] - t * lap - u0[j];
    sum += r * r;
  }
  free(u0);
  return sqrt(sum);
}

/* normalized_target_gradients (diffusion.hpp:132-145) */
int32_t gho_normalized_target_gradients(const gho_mesh* m, const double* u, double* h) {
  gho_face_gradient(m, u, h);
  int32_t zero = 0;
  for (int64_t f = 0; f < m->nf; ++f) {
    v3 g = v3_load(h, f);
    double norm = v3_norm(g);
    if (norm >= 1e-20) {
      v3_store(h, f, v3_div(v3_make(-g.x, -g.y, -g.z), norm));
    } else {
      v3_store(h, f, v3_make(0.0, 0.0, 0.0));
      ++zero;
    }
  }
  return zero;
}

/* ---------------------------------------------------------------- face ADMM */

static inline int32_t edge_face(const gho_mesh* m, int64_t e, int side) {
  int32_t h = m->edge_halfedges[2 * e + side];
  return h >= 0 ? h / 3 : -1;
}

static void record(gho_report* r, int32_t it, double primal, double dual) {
  if (!r) return;
  if (r->primal_history && it < r->history_capacity) r->primal_history[it] = primal;
  if (r->dual_history && it < r->history_capacity) r->dual_history[it] = dual;
  r->final_primal = primal;
  r->final_dual = dual;
  r->iterations = it + 1;
}

/* FaceAdmmSolver (grad_face.hpp:51-206) + admm_face_optimize (228-237) */
int gho_admm_face(const gho_mesh* m, const double* h, int32_t max_iterations, double eps1, double eps2, double mu,
                  double* g, gho_report* report) {
  if (max_iterations < 0 || !(eps1 > 0.0) || !(eps2 > 0.0) || !(mu > 0.0)) return 2;
  double t0 = now_seconds();
  const int64_t F = m->nf, NI = m->ni;
  if (report) {
    report->iterations = 0;
    report->converged = 0;
    report->final_primal = report->final_dual = 0.0;
    report->state_bytes_formula = (6 * (uint64_t)F + 15 * (uint64_t)NI) * 8; /* 217-223 */
  }
  double* y1 = (double*)malloc(sizeof(double) * (3 * NI + 3));
  double* y2 = (double*)malloc(sizeof(double) * (3 * NI + 3));
  double* l1 = (double*)calloc((size_t)(3 * NI + 3), sizeof(double));
  double* l2 = (double*)calloc((size_t)(3 * NI + 3), sizeof(double));
  double* edir = (double*)malloc(sizeof(double) * (3 * NI + 3));
  double* gprev = (double*)malloc(sizeof(double) * (3 * F + 3));
  double* se = (double*)malloc(sizeof(double) * (NI + 1));
  double* sf = (double*)malloc(sizeof(double) * (F + 1));
  memcpy(g, h, sizeof(double) * 3 * F);
  /* ctor (65-89) */
  double scale2 = 0.0;
  for (int64_t i = 0; i < NI; ++i) {
    int32_t e = m->interior_edges[i];
    v3_store(edir, i, v3_normalized(edge_vector(m, e)));
    int32_t f1 = edge_face(m, e, 0), f2 = edge_face(m, e, 1);
    v3_store(y1, i, v3_load(h, f1));
    v3_store(y2, i, v3_load(h, f2));
    scale2 += m->face_area[f1] + m->face_area[f2];
  }
  const double scale = sqrt(scale2);

  for (int32_t it = 0; it < max_iterations; ++it) {
    /* Y update (126-137) with y_update_edge (31-36) */
    for (int64_t i = 0; i < NI; ++i) {
      int32_t e = m->interior_edges[i];
      int32_t f1 = edge_face(m, e, 0), f2 = edge_face(m, e, 1);
      double a1 = m->face_area[f1], a2 = m->face_area[f2];
      v3 q1 = v3_sub(v3_load(g, f1), v3_div(v3_load(l1, i), mu * sqrt(a1)));
      v3 q2 = v3_sub(v3_load(g, f2), v3_div(v3_load(l2, i), mu * sqrt(a2)));
      v3 ed = v3_load(edir, i);
      double mismatch = v3_dot(ed, v3_sub(q2, q1));
      v3 shift = v3_make(ed.x * mismatch, ed.y * mismatch, ed.z * mismatch);
      v3_store(y1, i, v3_add(q1, v3_scale(a2 / (a1 + a2), shift)));
      v3_store(y2, i, v3_sub(q2, v3_scale(a1 / (a1 + a2), shift)));
    }
    /* G update (139-155) */
    memcpy(gprev, g, sizeof(double) * 3 * F);
    for (int64_t f = 0; f < F; ++f) {
      double alpha = sqrt(m->face_area[f]);
      v3 sum = v3_make(0.0, 0.0, 0.0);
      int count = 0;
      for (int k = 0; k < 3; ++k) {
        int32_t e = m->halfedge_edge[3 * f + k];
        int32_t i = m->interior_edge_index[e];
        if (i < 0) continue;
        int first = edge_face(m, e, 0) == f;
        v3 yk = v3_load(first ? y1 : y2, i);
        v3 lk = v3_load(first ? l1 : l2, i);
        sum = v3_add(sum, v3_add(yk, v3_div(lk, mu * alpha)));
        ++count;
      }
      v3 hf = v3_load(h, f);
      v3_store(g, f, v3_div(v3_add(v3_scale(2.0, hf), v3_scale(mu, sum)), 2.0 + mu * (double)count));
    }
    /* lambda update + primal rows (158-168) */
    for (int64_t i = 0; i < NI; ++i) {
      int32_t e = m->interior_edges[i];
      int32_t f1 = edge_face(m, e, 0), f2 = edge_face(m, e, 1);
      v3 r1 = v3_scale(sqrt(m->face_area[f1]), v3_sub(v3_load(y1, i), v3_load(g, f1)));
      v3 r2 = v3_scale(sqrt(m->face_area[f2]), v3_sub(v3_load(y2, i), v3_load(g, f2)));
      v3_store(l1, i, v3_add(v3_load(l1, i), v3_scale(mu, r1)));
      v3_store(l2, i, v3_add(v3_load(l2, i), v3_scale(mu, r2)));
      se[i] = v3_sqnorm(r1) + v3_sqnorm(r2);
    }
    double ps = 0.0;
    for (int64_t i = 0; i < NI; ++i) ps += se[i];
    const double primal = sqrt(ps);
    /* dual (170-171, 104-111) */
    for (int64_t f = 0; f < F; ++f) {
      v3 d = v3_sub(v3_load(g, f), v3_load(gprev, f));
      int deg = 0;
      for (int k = 0; k < 3; ++k)
        if (m->interior_edge_index[m->halfedge_edge[3 * f + k]] >= 0) ++deg;
      sf[f] = (double)deg * m->face_area[f] * v3_sqnorm(d);
    }
    double ds = 0.0;
    for (int64_t f = 0; f < F; ++f) ds += sf[f];
    const double dual = mu * sqrt(ds);
    record(report, it, primal, dual);
    if (primal <= scale * eps1 && dual <= scale * eps2) { /* 175-177 */
      if (report) report->converged = 1;
      break;
    }
  }
  if (report) {
    report->wall_seconds = now_seconds() - t0;
    /* allocated_bytes (grad_face.hpp:201-205): g, targets, y1, y2, l1, l2, edge_dir */
    report->state_bytes_allocated = (2 * (uint64_t)F + 5 * (uint64_t)NI) * 24;
  }
  free(y1); free(y2); free(l1); free(l2); free(edir); free(gprev); free(se); free(sf);
  return 0;
}

/* ---------------------------------------------------------------- edge ADMM */

/* EdgeAdmmSolver (grad_edge.hpp:57-198) + admm_edge_optimize (207-216) */
int gho_admm_edge(const gho_mesh* m, const double* h, int32_t max_iterations, double eps1, double eps2, double mu,
                  double* x, gho_report* report) {
  if (max_iterations < 0 || !(eps1 > 0.0) || !(eps2 > 0.0) || !(mu > 0.0)) return 2;
  double t0 = now_seconds();
  const int64_t F = m->nf, E = m->ne;
  if (report) {
    report->iterations = 0;
    report->converged = 0;
    report->final_primal = report->final_dual = 0.0;
    report->state_bytes_formula = (6 * (uint64_t)F + 2 * (uint64_t)E) * 8 + 3 * (uint64_t)F;
  }
  double* w = (double*)malloc(sizeof(double) * (3 * F + 1));
  double* lam = (double*)calloc((size_t)(3 * F + 1), sizeof(double));
  double* sgn = (double*)malloc(sizeof(double) * (3 * F + 1));
  double* tsum = (double*)calloc((size_t)E + 1, sizeof(double));
  double* xprev = (double*)malloc(sizeof(double) * (E + 1));
  double* sf = (double*)malloc(sizeof(double) * (F + 1));
  double* se = (double*)malloc(sizeof(double) * (E + 1));
  const double scale = sqrt(3.0 * (double)F);
  /* ctor (72-98): targets z (19-26), signs (mesh.hpp:81-83) */
  for (int64_t f = 0; f < F; ++f) {
    v3 hf = v3_load(h, f);
    for (int k = 0; k < 3; ++k) {
      int64_t hh = 3 * f + k;
      int32_t e = m->halfedge_edge[hh];
      double z = v3_dot(hf, edge_vector(m, e));
      w[hh] = z;
      sgn[hh] = he_tail(m, hh) == m->edge_vertices[2 * e] ? 1.0 : -1.0;
      tsum[e] += z;
    }
  }
  for (int64_t e = 0; e < E; ++e) {
    int deg = (m->edge_halfedges[2 * e] >= 0 && m->edge_halfedges[2 * e + 1] >= 0) ? 2 : 1;
    x[e] = tsum[e] / (double)deg;
  }

  for (int32_t it = 0; it < max_iterations; ++it) {
    /* W (131-141) */
    for (int64_t f = 0; f < F; ++f) {
      double dot = 0.0, v[3];
      for (int k = 0; k < 3; ++k) {
        int64_t hh = 3 * f + k;
        v[k] = x[m->halfedge_edge[hh]] - lam[hh] / mu;
        dot += sgn[hh] * v[k];
      }
      double shift = dot / 3.0;
      for (int k = 0; k < 3; ++k) w[3 * f + k] = v[k] - shift * sgn[3 * f + k];
    }
    /* X (143-149) */
    for (int64_t e = 0; e < E; ++e) {
      xprev[e] = x[e];
      double sum = tsum[e];
      for (int s = 0; s < 2; ++s) {
        int32_t hh = m->edge_halfedges[2 * e + s];
        if (hh >= 0) sum += lam[hh] + mu * w[hh];
      }
      int deg = (m->edge_halfedges[2 * e] >= 0 && m->edge_halfedges[2 * e + 1] >= 0) ? 2 : 1;
      x[e] = sum / ((double)deg * (1.0 + mu));
    }
    /* lambda + primal (151-158) */
    for (int64_t f = 0; f < F; ++f) {
      double sum = 0.0;
      for (int k = 0; k < 3; ++k) {
        int64_t hh = 3 * f + k;
        double r = w[hh] - x[m->halfedge_edge[hh]];
        lam[hh] += mu * r;
        sum += r * r;
      }
      sf[f] = sum;
    }
    double ps = 0.0;
    for (int64_t f = 0; f < F; ++f) ps += sf[f];
    const double primal = sqrt(ps);
    /* dual (160-164, 114-120) */
    for (int64_t e = 0; e < E; ++e) {
      double d = x[e] - xprev[e];
      int deg = (m->edge_halfedges[2 * e] >= 0 && m->edge_halfedges[2 * e + 1] >= 0) ? 2 : 1;
      se[e] = (double)deg * d * d;
    }
    double ds = 0.0;
    for (int64_t e = 0; e < E; ++e) ds += se[e];
    const double dual = mu * sqrt(ds);
    record(report, it, primal, dual);
    if (primal <= scale * eps1 && dual <= scale * eps2) {
      if (report) report->converged = 1;
      break;
    }
  }
  if (report) {
    report->wall_seconds = now_seconds() - t0;
    report->state_bytes_allocated = (2 * (uint64_t)E + 6 * (uint64_t)F) * 8 + 3 * (uint64_t)F;
  }
  free(w); free(lam); free(sgn); free(tsum); free(xprev); free(sf); free(se);
  return 0;
}

/* ---------------------------------------------------------------- integration */

/* run_levels + integrate_face_gradients (integrate.hpp:19-59) */
void gho_integrate_face(const gho_mesh* m, const gho_levels* l, const double* g, double* d) {
  for (int64_t v = 0; v < m->nv; ++v) d[v] = INFINITY;
  for (int32_t i = l->offsets[0]; i < l->offsets[1]; ++i) d[l->order[i]] = 0.0;
  for (int32_t li = 1; li < l->nlev; ++li) {
    for (int32_t i = l->offsets[li]; i < l->offsets[li + 1]; ++i) {
      int32_t v = l->order[i];
      int32_t parent = l->parent_of_vertex[v];
      int32_t e = edge_between(m, parent, v);
      v3 step = v3_sub(v3_load(m->positions, v), v3_load(m->positions, parent));
      double sum = 0.0;
      int count = 0;
      for (int s = 0; s < 2; ++s) {
        int32_t hh = m->edge_halfedges[2 * e + s];
        if (hh < 0) continue;
        sum += v3_dot(v3_load(g, hh / 3), step);
        ++count;
      }
      d[v] = d[parent] + sum / (double)count;
    }
  }
}

/* integrate_edge_differences (integrate.hpp:64-75) */
void gho_integrate_edge(const gho_mesh* m, const gho_levels* l, const double* x, double* d) {
  for (int64_t v = 0; v < m->nv; ++v) d[v] = INFINITY;
  for (int32_t i = l->offsets[0]; i < l->offsets[1]; ++i) d[l->order[i]] = 0.0;
  for (int32_t li = 1; li < l->nlev; ++li) {
    for (int32_t i = l->offsets[li]; i < l->offsets[li + 1]; ++i) {
      int32_t v = l->order[i];
      int32_t parent = l->parent_of_vertex[v];
      int32_t e = edge_between(m, parent, v);
      double sigma = m->edge_vertices[2 * e] == parent ? 1.0 : -1.0;
      d[v] = d[parent] + sigma * x[e];
    }
  }
}

/* field_hash (report.hpp:145-153): FNV-1a over the raw bytes */
uint64_t gho_field_hash(const double* values, int64_t n) {
  uint64_t h = 1469598103934665603ull;
  const unsigned char* bytes = (const unsigned char*)values;
  for (int64_t i = 0; i < n * (int64_t)sizeof(double); ++i) {
    h ^= bytes[i];
    h *= 1099511628211ull;
  }
  return h;
}
