/*
 * parplan_oracle.c — plain-C restatement of the reference planner.
 *
 * TEST INFRASTRUCTURE ONLY (see parplan_oracle.h).  This is the checker the
 * CUDA product is compared against; the product never calls it.
 *
 * Citations are relative to /root/reference/proj/include/parplan/.
 */
#include "parplan_oracle.h"

#include <float.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* errors                                                                   */
/* ------------------------------------------------------------------------ */

static _Thread_local char g_err[512];

static void set_err(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

const char *orc_error(void) { return g_err; }
int orc_kind(void) { return 0; }

static void *xcalloc(size_t n, size_t s) {
  void *p = calloc(n ? n : 1, s ? s : 1);
  if (!p) {
    fprintf(stderr, "oracle: out of memory\n");
    abort();
  }
  return p;
}

/* ------------------------------------------------------------------------ */
/* mt19937_64 — the generator std::mt19937_64 specifies (oracle.hpp:129)    */
/* ------------------------------------------------------------------------ */

#define MT_N 312
#define MT_M 156
typedef struct {
  uint64_t s[MT_N];
  int i;
} mt64;

static void mt_seed(mt64 *m, uint64_t seed) {
  m->s[0] = seed;
  for (int k = 1; k < MT_N; ++k) m->s[k] = 6364136223846793005ULL * (m->s[k - 1] ^ (m->s[k - 1] >> 62)) + (uint64_t)k;
  m->i = MT_N;
}

static uint64_t mt_next(mt64 *m) {
  if (m->i >= MT_N) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
    for (int k = 0; k < MT_N; ++k) {
      uint64_t y = (m->s[k] & UM) | (m->s[(k + 1) % MT_N] & LM);
      m->s[k] = m->s[(k + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
    }
    m->i = 0;
  }
  uint64_t x = m->s[m->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* ------------------------------------------------------------------------ */
/* instance                                                                 */
/* ------------------------------------------------------------------------ */

typedef struct {
  int n;
  int cap;
  int *v;
} ivec;

static void iv_push(ivec *a, int x) {
  if (a->n == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 4;
    a->v = (int *)realloc(a->v, (size_t)a->cap * sizeof(int));
  }
  a->v[a->n++] = x;
}
static void iv_erase(ivec *a, int x) { /* planner.hpp:229-236: erase first occurrence, keep order */
  for (int k = 0; k < a->n; ++k)
    if (a->v[k] == x) {
      memmove(a->v + k, a->v + k + 1, (size_t)(a->n - k - 1) * sizeof(int));
      --a->n;
      return;
    }
}

typedef struct {
  int type; /* 0 node, 1 edge */
  int removed, e1, e2, ne, src, dst;
  int nu, nv;
  int32_t *argmin; /* [nu*nv] */
} orc_rec;

typedef struct {
  int id, src, dst, alive;
  int nu, nv;
  double *t; /* [nu*nv] */
} orc_redge;

struct orc_instance {
  /* graph */
  int nl, ne;
  int64_t batch;
  int *kind;
  int64_t *params; /* nl*7 */
  char **ids;
  int *esrc, *edst, *epos;
  ivec *in_e, *out_e;
  int *topo, *rank;
  int64_t *shape; /* nl*4 */
  /* tables */
  int have_tables;
  int *ncfg;
  int64_t **cat; /* per layer, 4*ncfg */
  double **node, **compute, **sync;
  double **xfer; /* per edge, ncfg[src]*ncfg[dst] */
  /* reduced graph */
  int reduced;
  int *alive;
  int n_redges, cap_redges;
  orc_redge *redges;
  ivec *rin, *rout;
  int n_log, cap_log;
  orc_rec *log;
};

static void free_reduced(orc_instance *g) {
  if (!g->reduced) return;
  for (int k = 0; k < g->n_redges; ++k) free(g->redges[k].t);
  free(g->redges);
  for (int l = 0; l < g->nl; ++l) {
    free(g->rin[l].v);
    free(g->rout[l].v);
  }
  free(g->rin);
  free(g->rout);
  for (int k = 0; k < g->n_log; ++k) free(g->log[k].argmin);
  free(g->log);
  free(g->alive);
  g->reduced = 0;
  g->n_redges = g->cap_redges = g->n_log = g->cap_log = 0;
  g->redges = NULL;
  g->log = NULL;
}

static void free_tables(orc_instance *g) {
  if (!g->have_tables) return;
  for (int l = 0; l < g->nl; ++l) {
    free(g->cat[l]);
    free(g->node[l]);
    free(g->compute[l]);
    free(g->sync[l]);
  }
  for (int e = 0; e < g->ne; ++e) free(g->xfer[e]);
  free(g->ncfg);
  free(g->cat);
  free(g->node);
  free(g->compute);
  free(g->sync);
  free(g->xfer);
  g->have_tables = 0;
}

void orc_free(orc_instance *g) {
  if (!g) return;
  free_reduced(g);
  free_tables(g);
  for (int l = 0; l < g->nl; ++l) {
    free(g->ids[l]);
    free(g->in_e[l].v);
    free(g->out_e[l].v);
  }
  free(g->ids);
  free(g->in_e);
  free(g->out_e);
  free(g->kind);
  free(g->params);
  free(g->esrc);
  free(g->edst);
  free(g->epos);
  free(g->topo);
  free(g->rank);
  free(g->shape);
  free(g);
}

/* ------------------------------------------------------------------------ */
/* graph creation (graph.hpp:263-360) and shape inference (:362-435)        */
/* ------------------------------------------------------------------------ */

static int64_t conv_out(int64_t in, int64_t k, int64_t s, int64_t p) { return (in + 2 * p - k) / s + 1; } /* :257-259 */

static int validate_params(const orc_instance *g, int l) { /* graph.hpp:233-255 */
  const int64_t *p = g->params + 7 * l;
  const char *id = g->ids[l];
  switch (g->kind[l]) {
  case ORC_CONV:
    if (p[0] < 1) return set_err("layer '%s': out_channels must be >= 1", id), 1;
    if (p[1] < 1 || p[2] < 1 || p[3] < 1 || p[4] < 1) return set_err("layer '%s': kernel/stride must be >= 1", id), 1;
    if (p[5] < 0 || p[6] < 0) return set_err("layer '%s': padding must be >= 0", id), 1;
    break;
  case ORC_POOL:
    if (p[0] < 1 || p[1] < 1 || p[2] < 1 || p[3] < 1) return set_err("layer '%s': kernel/stride must be >= 1", id), 1;
    if (p[4] < 0 || p[5] < 0) return set_err("layer '%s': padding must be >= 0", id), 1;
    break;
  case ORC_FC:
    if (p[0] < 1) return set_err("layer '%s': out_channels must be >= 1", id), 1;
    break;
  case ORC_INPUT:
    if (p[0] < 1 || p[1] < 1 || p[2] < 1) return set_err("layer '%s': input extents must be >= 1", id), 1;
    break;
  default:
    break;
  }
  return 0;
}

static int infer_shapes(orc_instance *g) { /* graph.hpp:362-435, in topo order */
  for (int r = 0; r < g->nl; ++r) {
    const int v = g->topo[r];
    const int64_t *p = g->params + 7 * v;
    int64_t *o = g->shape + 4 * v;
    const int64_t *in = g->in_e[v].n ? g->shape + 4 * g->esrc[g->in_e[v].v[0]] : NULL;
    switch (g->kind[v]) {
    case ORC_INPUT:
      o[0] = g->batch, o[1] = p[0], o[2] = p[1], o[3] = p[2];
      break;
    case ORC_CONV:
    case ORC_POOL: {
      const int conv = g->kind[v] == ORC_CONV;
      const int64_t *w = conv ? p + 1 : p; /* kh, kw, sh, sw, ph, pw */
      o[0] = in[0];
      o[1] = conv ? p[0] : in[1];
      o[2] = conv_out(in[2], w[0], w[2], w[4]);
      o[3] = conv_out(in[3], w[1], w[3], w[5]);
      if (o[2] < 1 || o[3] < 1)
        return set_err("layer '%s': non-positive inferred extent (%lld, %lld, %lld, %lld)", g->ids[v], (long long)o[0],
                       (long long)o[1], (long long)o[2], (long long)o[3]),
               1;
      break;
    }
    case ORC_FC:
      o[0] = in[0], o[1] = p[0], o[2] = 1, o[3] = 1;
      break;
    case ORC_FLATTEN:
      o[0] = in[0], o[1] = in[1] * in[2] * in[3], o[2] = 1, o[3] = 1;
      break;
    case ORC_CONCAT: {
      const int axis = (int)p[0];
      memcpy(o, in, 4 * sizeof(int64_t));
      for (int k = 1; k < g->in_e[v].n; ++k) {
        const int64_t *s = g->shape + 4 * g->esrc[g->in_e[v].v[k]];
        for (int d = 0; d < 4; ++d)
          if (d != axis && s[d] != o[d]) return set_err("layer '%s': concat extent mismatch", g->ids[v]), 1;
        o[axis] += s[axis];
      }
      break;
    }
    case ORC_SOFTMAX:
      memcpy(o, in, 4 * sizeof(int64_t));
      break;
    }
  }
  return 0;
}

orc_instance *orc_graph(int nl, int ne, int64_t batch, const int32_t *kind, const int64_t *params, const int32_t *esrc,
                        const int32_t *edst, const char *const *ids) {
  g_err[0] = 0;
  if (batch < 1) return set_err("batch must be >= 1"), NULL;
  if (nl < 1) return set_err("graph needs at least one layer"), NULL;
  orc_instance *g = (orc_instance *)xcalloc(1, sizeof *g);
  g->nl = nl;
  g->ne = ne;
  g->batch = batch;
  g->kind = (int *)xcalloc((size_t)nl, sizeof(int));
  g->params = (int64_t *)xcalloc((size_t)nl * 7, sizeof(int64_t));
  g->ids = (char **)xcalloc((size_t)nl, sizeof(char *));
  g->in_e = (ivec *)xcalloc((size_t)nl, sizeof(ivec));
  g->out_e = (ivec *)xcalloc((size_t)nl, sizeof(ivec));
  g->esrc = (int *)xcalloc((size_t)ne, sizeof(int));
  g->edst = (int *)xcalloc((size_t)ne, sizeof(int));
  g->epos = (int *)xcalloc((size_t)ne, sizeof(int));
  g->topo = (int *)xcalloc((size_t)nl, sizeof(int));
  g->rank = (int *)xcalloc((size_t)nl, sizeof(int));
  g->shape = (int64_t *)xcalloc((size_t)nl * 4, sizeof(int64_t));
  for (int l = 0; l < nl; ++l) {
    g->kind[l] = kind[l];
    memcpy(g->params + 7 * l, params + 7 * l, 7 * sizeof(int64_t));
    char buf[32];
    snprintf(buf, sizeof buf, "n%d", l);
    const char *id = ids ? ids[l] : buf;
    g->ids[l] = (char *)xcalloc(strlen(id) + 1, 1);
    strcpy(g->ids[l], id);
  }
  /* duplicate ids + params (graph.hpp:281-289) */
  for (int l = 0; l < nl; ++l) {
    if (!g->ids[l][0]) return set_err("layer at position %d has an empty id", l), orc_free(g), NULL;
    for (int k = 0; k < l; ++k)
      if (!strcmp(g->ids[k], g->ids[l])) return set_err("duplicate layer id '%s'", g->ids[l]), orc_free(g), NULL;
    if (validate_params(g, l)) return orc_free(g), NULL;
  }
  /* edges in creation order; dst_input_pos = running count per dst (graph.hpp:291-318) */
  for (int e = 0; e < ne; ++e) {
    if (esrc[e] < 0 || esrc[e] >= nl || edst[e] < 0 || edst[e] >= nl)
      return set_err("edge %d references an undeclared layer", e), orc_free(g), NULL;
    if (e && edst[e] < edst[e - 1]) return set_err("edges must be listed in destination order"), orc_free(g), NULL;
    g->esrc[e] = esrc[e];
    g->edst[e] = edst[e];
    g->epos[e] = g->in_e[edst[e]].n;
    iv_push(&g->out_e[esrc[e]], e);
    iv_push(&g->in_e[edst[e]], e);
  }
  for (int l = 0; l < nl; ++l) { /* arity (graph.hpp:294-303) */
    const int n = g->in_e[l].n;
    if (g->kind[l] == ORC_INPUT && n) return set_err("input layer '%s' cannot have inputs", g->ids[l]), orc_free(g), NULL;
    if (g->kind[l] == ORC_CONCAT && n < 2)
      return set_err("concat layer '%s' needs at least 2 inputs", g->ids[l]), orc_free(g), NULL;
    if (g->kind[l] != ORC_INPUT && g->kind[l] != ORC_CONCAT && n != 1)
      return set_err("layer '%s' must have exactly 1 input, got %d", g->ids[l], n), orc_free(g), NULL;
  }
  /* Kahn with a min-index priority queue (graph.hpp:321-349); n is small so a
   * linear scan of the ready set is the same order as the binary heap. */
  int *indeg = (int *)xcalloc((size_t)nl, sizeof(int));
  char *ready = (char *)xcalloc((size_t)nl, 1);
  for (int e = 0; e < ne; ++e) ++indeg[g->edst[e]];
  for (int l = 0; l < nl; ++l) ready[l] = indeg[l] == 0;
  int nt = 0;
  for (;;) {
    int v = -1;
    for (int l = 0; l < nl; ++l)
      if (ready[l]) {
        v = l;
        break;
      }
    if (v < 0) break;
    ready[v] = 0;
    g->topo[nt++] = v;
    for (int k = 0; k < g->out_e[v].n; ++k) {
      const int d = g->edst[g->out_e[v].v[k]];
      if (--indeg[d] == 0) ready[d] = 1;
    }
  }
  if (nt != nl) {
    int stuck = 0;
    for (int l = 0; l < nl; ++l)
      if (indeg[l] > 0) {
        stuck = l;
        break;
      }
    set_err("graph contains a cycle through layer '%s'", g->ids[stuck]);
    free(indeg), free(ready), orc_free(g);
    return NULL;
  }
  free(indeg);
  free(ready);
  for (int r = 0; r < nl; ++r) g->rank[g->topo[r]] = r;
  for (int l = 0; l < nl; ++l) /* graph.hpp:352-357 */
    if (!g->in_e[l].n && g->kind[l] != ORC_INPUT)
      return set_err("layer '%s' has no inputs but is not an input layer", g->ids[l]), orc_free(g), NULL;
  if (infer_shapes(g)) return orc_free(g), NULL;
  return g;
}

/* ------------------------------------------------------------------------ */
/* builtin models (models.hpp:61-131)                                       */
/* ------------------------------------------------------------------------ */

typedef struct {
  int nl, ne, capl, cape;
  int32_t *kind;
  int64_t *params;
  char **ids;
  int32_t *esrc, *edst;
} builder;

static int b_find(const builder *b, const char *id) {
  for (int l = b->nl - 1; l >= 0; --l)
    if (!strcmp(b->ids[l], id)) return l;
  return -1;
}

static int b_add(builder *b, const char *id, int kind, const int64_t *p, int nin, const int *in) {
  if (b->nl == b->capl) {
    b->capl = b->capl ? 2 * b->capl : 16;
    b->kind = (int32_t *)realloc(b->kind, (size_t)b->capl * sizeof(int32_t));
    b->params = (int64_t *)realloc(b->params, (size_t)b->capl * 7 * sizeof(int64_t));
    b->ids = (char **)realloc(b->ids, (size_t)b->capl * sizeof(char *));
  }
  const int l = b->nl++;
  b->kind[l] = kind;
  memset(b->params + 7 * l, 0, 7 * sizeof(int64_t));
  if (p) memcpy(b->params + 7 * l, p, 7 * sizeof(int64_t));
  b->ids[l] = (char *)xcalloc(strlen(id) + 1, 1);
  strcpy(b->ids[l], id);
  for (int k = 0; k < nin; ++k) {
    if (b->ne == b->cape) {
      b->cape = b->cape ? 2 * b->cape : 16;
      b->esrc = (int32_t *)realloc(b->esrc, (size_t)b->cape * sizeof(int32_t));
      b->edst = (int32_t *)realloc(b->edst, (size_t)b->cape * sizeof(int32_t));
    }
    b->esrc[b->ne] = in[k];
    b->edst[b->ne] = l;
    ++b->ne;
  }
  return l;
}

static orc_instance *b_build(builder *b, int64_t batch) {
  orc_instance *g = orc_graph(b->nl, b->ne, batch, b->kind, b->params, b->esrc, b->edst, (const char *const *)b->ids);
  for (int l = 0; l < b->nl; ++l) free(b->ids[l]);
  free(b->ids), free(b->kind), free(b->params), free(b->esrc), free(b->edst);
  return g;
}

static int add_conv(builder *b, const char *id, int64_t oc, int64_t k, int64_t s, int64_t p, int in) {
  int64_t q[7] = {oc, k, k, s, s, p, p};
  return b_add(b, id, ORC_CONV, q, 1, &in);
}
static int add_pool(builder *b, const char *id, int64_t k, int64_t s, int64_t p, int in) {
  int64_t q[7] = {k, k, s, s, p, p, 0};
  return b_add(b, id, ORC_POOL, q, 1, &in);
}
static int add_fc(builder *b, const char *id, int64_t oc, int in) {
  int64_t q[7] = {oc, 0, 0, 0, 0, 0, 0};
  return b_add(b, id, ORC_FC, q, 1, &in);
}
static int add_input(builder *b, const char *id, int64_t c, int64_t h, int64_t w) {
  int64_t q[7] = {c, h, w, 0, 0, 0, 0};
  return b_add(b, id, ORC_INPUT, q, 0, NULL);
}

orc_instance *orc_builtin(const char *name, int64_t batch) {
  builder b;
  memset(&b, 0, sizeof b);
  g_err[0] = 0;
  if (!strcmp(name, "lenet5")) { /* models.hpp:61-70 */
    int x = add_input(&b, "input", 1, 32, 32);
    x = add_conv(&b, "conv1", 6, 5, 1, 0, x);
    x = add_pool(&b, "pool1", 2, 2, 0, x);
    x = add_conv(&b, "conv2", 16, 5, 1, 0, x);
    x = add_pool(&b, "pool2", 2, 2, 0, x);
    add_fc(&b, "fc1", 10, x);
  } else if (!strcmp(name, "alexnet")) { /* models.hpp:73-87 */
    int x = add_input(&b, "input", 3, 224, 224);
    x = add_conv(&b, "conv1", 96, 11, 4, 2, x);
    x = add_pool(&b, "pool1", 3, 2, 0, x);
    x = add_conv(&b, "conv2", 256, 5, 1, 2, x);
    x = add_pool(&b, "pool2", 3, 2, 0, x);
    x = add_conv(&b, "conv3", 384, 3, 1, 1, x);
    x = add_conv(&b, "conv4", 384, 3, 1, 1, x);
    x = add_conv(&b, "conv5", 256, 3, 1, 1, x);
    x = add_pool(&b, "pool3", 3, 2, 0, x);
    x = add_fc(&b, "fc1", 4096, x);
    add_fc(&b, "fc2", 1000, x);
  } else if (!strcmp(name, "vgg16")) { /* models.hpp:91-107 */
    static const int widths[5] = {64, 128, 256, 512, 512}, convs[5] = {2, 2, 3, 3, 3};
    int x = add_input(&b, "input", 3, 224, 224);
    char id[32];
    for (int bi = 0; bi < 5; ++bi) {
      for (int ci = 0; ci < convs[bi]; ++ci) {
        snprintf(id, sizeof id, "conv%d_%d", bi + 1, ci + 1);
        x = add_conv(&b, id, widths[bi], 3, 1, 1, x);
      }
      snprintf(id, sizeof id, "pool%d", bi + 1);
      x = add_pool(&b, id, 2, 2, 0, x);
    }
    x = add_fc(&b, "fc1", 4096, x);
    add_fc(&b, "fc2", 1000, x);
  } else if (!strncmp(name, "inception_chain", 15)) { /* models.hpp:113-131, :150-160 */
    int modules = 12;
    if (name[15] == '(') {
      char *end = NULL;
      long m = strtol(name + 16, &end, 10);
      if (!end || end == name + 16 || strcmp(end, ")")) return set_err("invalid module count in '%s'", name), NULL;
      modules = (int)m;
    } else if (name[15]) {
      return set_err("unknown model '%s' (builtins: lenet5, alexnet, vgg16, inception_chain)", name), NULL;
    }
    if (modules < 1) return set_err("inception_chain: module count must be >= 1"), NULL;
    int x = add_input(&b, "input", 192, 35, 35);
    char id[32];
    for (int m = 1; m <= modules; ++m) {
#define MID(s) (snprintf(id, sizeof id, "m%d_%s", m, s), id)
      int b1 = add_conv(&b, MID("b1"), 64, 1, 1, 0, x);
      int b2 = add_conv(&b, MID("b2a"), 48, 1, 1, 0, x);
      b2 = add_conv(&b, MID("b2b"), 64, 5, 1, 2, b2);
      int b3 = add_conv(&b, MID("b3a"), 64, 1, 1, 0, x);
      b3 = add_conv(&b, MID("b3b"), 96, 3, 1, 1, b3);
      b3 = add_conv(&b, MID("b3c"), 96, 3, 1, 1, b3);
      int b4 = add_pool(&b, MID("b4p"), 3, 1, 1, x);
      b4 = add_conv(&b, MID("b4c"), 64, 1, 1, 0, b4);
      int ins[4] = {b1, b2, b3, b4};
      int64_t q[7] = {1, 0, 0, 0, 0, 0, 0};
      x = b_add(&b, MID("join"), ORC_CONCAT, q, 4, ins);
#undef MID
    }
  } else {
    return set_err("unknown model '%s' (builtins: lenet5, alexnet, vgg16, inception_chain)", name), NULL;
  }
  (void)b_find;
  return b_build(&b, batch);
}

/* ------------------------------------------------------------------------ */
/* config enumeration (partition.hpp:140-204)                               */
/* ------------------------------------------------------------------------ */

static void parallel_dims(int kind, const int64_t *shape, int dims[4]) { /* partition.hpp:140-156 */
  for (int d = 0; d < 4; ++d) dims[d] = 0;
  if (kind == ORC_CONV || kind == ORC_POOL) {
    for (int d = 0; d < 4; ++d) dims[d] = 1;
  } else if (kind == ORC_FC || kind == ORC_SOFTMAX) {
    dims[0] = dims[1] = 1;
  } else {
    for (int d = 0; d < 4; ++d) dims[d] = shape[d] > 1;
  }
}

int orc_enumerate_configs(int kind, const int64_t *shape, int device_count, int64_t *out, int cap) {
  if (device_count < 1) return set_err("enumerate_configs: need at least one device"), -1;
  int dims[4];
  parallel_dims(kind, shape, dims);
  const int64_t D = device_count;
  int64_t ch[4][64];
  int nch[4];
  for (int d = 0; d < 4; ++d) { /* divisors_up_to (:160-166) */
    nch[d] = 0;
    if (!dims[d]) {
      ch[d][nch[d]++] = 1;
      continue;
    }
    const int64_t lim = shape[d] < D ? shape[d] : D;
    for (int64_t x = 1; x <= lim; ++x)
      if (shape[d] % x == 0 && nch[d] < 64) ch[d][nch[d]++] = x;
  }
  int n = 0;
  for (int a = 0; a < nch[0]; ++a)
    for (int b = 0; b < nch[1]; ++b) {
      if (ch[0][a] * ch[1][b] > D) break;
      for (int c = 0; c < nch[2]; ++c) {
        if (ch[0][a] * ch[1][b] * ch[2][c] > D) break;
        for (int w = 0; w < nch[3]; ++w) {
          if (ch[0][a] * ch[1][b] * ch[2][c] * ch[3][w] > D) break;
          if (n < cap) {
            out[4 * n + 0] = ch[0][a], out[4 * n + 1] = ch[1][b];
            out[4 * n + 2] = ch[2][c], out[4 * n + 3] = ch[3][w];
          }
          ++n;
        }
      }
    }
  return n;
}

/* ------------------------------------------------------------------------ */
/* regions (partition.hpp:85-120, :213-350)                                 */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t lo[4], hi[4];
} region;

static int64_t reg_volume(const region *r) {
  int64_t v = 1;
  for (int d = 0; d < 4; ++d) v *= r->hi[d] > r->lo[d] ? r->hi[d] - r->lo[d] : 0;
  return v;
}

static region reg_intersect(const region *a, const region *b) {
  region r;
  for (int d = 0; d < 4; ++d) {
    r.lo[d] = a->lo[d] > b->lo[d] ? a->lo[d] : b->lo[d];
    r.hi[d] = a->hi[d] < b->hi[d] ? a->hi[d] : b->hi[d];
    if (r.hi[d] < r.lo[d]) r.hi[d] = r.lo[d];
  }
  return r;
}

static int64_t cfg_total(const int64_t *c) { return c[0] * c[1] * c[2] * c[3]; }

/* partition.hpp:213-232: W fastest, equal contiguous pieces */
static region owned(const int64_t *shape, const int64_t *cfg, int64_t part) {
  region r;
  int64_t rest = part;
  for (int d = 3; d >= 0; --d) {
    const int64_t idx = rest % cfg[d];
    rest /= cfg[d];
    const int64_t piece = shape[d] / cfg[d];
    r.lo[d] = idx * piece;
    r.hi[d] = r.lo[d] + piece;
  }
  return r;
}

int orc_owned_region(const int64_t *shape, const int64_t *config, int64_t part, int64_t *out8) {
  if (part < 0 || part >= cfg_total(config)) return set_err("owned_region: partition index out of range"), 1;
  region r = owned(shape, config, part);
  memcpy(out8, r.lo, 4 * sizeof(int64_t));
  memcpy(out8 + 4, r.hi, 4 * sizeof(int64_t));
  return 0;
}

static void window(region *req, const region *own, int d, int64_t k, int64_t s, int64_t p, int64_t ext) { /* :236-245 */
  const int64_t lo = own->lo[d] * s - p;
  const int64_t hi = (own->hi[d] - 1) * s - p + k;
  req->lo[d] = lo > 0 ? lo : 0;
  req->hi[d] = hi < ext ? hi : ext;
  if (req->hi[d] < req->lo[d]) req->hi[d] = req->lo[d];
}

static void flat_box(region *req, int64_t flo, int64_t fhi, int64_t H, int64_t W) { /* :249-273 */
  const int64_t plane = H * W;
  const int64_t clo = flo / plane, chi = (fhi - 1) / plane;
  req->lo[1] = clo;
  req->hi[1] = chi + 1;
  if (clo != chi) {
    req->lo[2] = 0, req->hi[2] = H, req->lo[3] = 0, req->hi[3] = W;
    return;
  }
  const int64_t rlo = (flo % plane) / W, rhi = ((fhi - 1) % plane) / W;
  req->lo[2] = rlo;
  req->hi[2] = rhi + 1;
  if (rlo != rhi) {
    req->lo[3] = 0, req->hi[3] = W;
    return;
  }
  req->lo[3] = flo % W;
  req->hi[3] = (fhi - 1) % W + 1;
}

static region required(const orc_instance *g, int e, const int64_t *dcfg, int64_t part) { /* :283-350 */
  const int dst = g->edst[e];
  const int64_t *oshape = g->shape + 4 * dst;
  const int64_t *ishape = g->shape + 4 * g->esrc[e];
  const int64_t *p = g->params + 7 * dst;
  const region own = owned(oshape, dcfg, part);
  region req;
  memset(&req, 0, sizeof req);
  req.lo[0] = own.lo[0];
  req.hi[0] = own.hi[0];
  switch (g->kind[dst]) {
  case ORC_CONV:
    req.lo[1] = 0, req.hi[1] = ishape[1];
    window(&req, &own, 2, p[1], p[3], p[5], ishape[2]);
    window(&req, &own, 3, p[2], p[4], p[6], ishape[3]);
    return req;
  case ORC_POOL:
    req.lo[1] = own.lo[1], req.hi[1] = own.hi[1];
    window(&req, &own, 2, p[0], p[2], p[4], ishape[2]);
    window(&req, &own, 3, p[1], p[3], p[5], ishape[3]);
    return req;
  case ORC_FC:
    req.lo[1] = 0, req.hi[1] = ishape[1];
    req.lo[2] = 0, req.hi[2] = ishape[2];
    req.lo[3] = 0, req.hi[3] = ishape[3];
    return req;
  case ORC_FLATTEN:
    flat_box(&req, own.lo[1], own.hi[1], ishape[2], ishape[3]);
    return req;
  case ORC_CONCAT: {
    const int A = (int)p[0];
    int64_t off = 0;
    for (int k = 0; k < g->in_e[dst].n; ++k) {
      const int sib = g->in_e[dst].v[k];
      if (g->epos[sib] == g->epos[e]) break;
      off += g->shape[4 * g->esrc[sib] + A];
    }
    region band = own;
    band.lo[A] = own.lo[A] > off ? own.lo[A] : off;
    band.hi[A] = own.hi[A] < off + ishape[A] ? own.hi[A] : off + ishape[A];
    if (band.hi[A] < band.lo[A]) band.hi[A] = band.lo[A];
    band.lo[A] -= off;
    band.hi[A] -= off;
    return band;
  }
  default: /* Softmax */
    return own;
  }
}

int orc_required_region(const orc_instance *g, int e, const int64_t *dcfg, int64_t part, int64_t *out8) {
  region r = required(g, e, dcfg, part);
  memcpy(out8, r.lo, 4 * sizeof(int64_t));
  memcpy(out8 + 4, r.hi, 4 * sizeof(int64_t));
  return 0;
}

/* ------------------------------------------------------------------------ */
/* cost model (cost.hpp:28-137)                                             */
/* ------------------------------------------------------------------------ */

static int64_t layer_flops(int kind, const int64_t *p, const int64_t *o, const int64_t *in) { /* :30-44 */
  switch (kind) {
  case ORC_CONV:
    return 2 * o[0] * o[1] * o[2] * o[3] * in[1] * p[1] * p[2];
  case ORC_POOL:
    return o[0] * o[1] * o[2] * o[3] * p[0] * p[1];
  case ORC_FC:
    return 2 * o[0] * (in[0] * in[1] * in[2] * in[3]) / in[0] * o[1];
  case ORC_SOFTMAX:
    return 5 * o[0] * o[1];
  default:
    return 0;
  }
}

static double param_bytes(int kind, const int64_t *p, const int64_t *o, const int64_t *in) { /* :46-55 */
  if (kind == ORC_CONV) return 4.0 * (double)o[1] * (double)in[1] * (double)p[1] * (double)p[2];
  if (kind == ORC_FC) return 4.0 * (double)((in[0] * in[1] * in[2] * in[3]) / in[0]) * (double)o[1];
  return 0.0;
}

static double compute_cost(int kind, const int64_t *p, const int64_t *o, const int64_t *in, const int64_t *cfg,
                           const double *rates) { /* :60-72 */
  const int64_t f = layer_flops(kind, p, o, in);
  if (f == 0) return 0.0;
  const int64_t tot = cfg_total(cfg);
  double slow = rates[0];
  for (int64_t q = 1; q < tot; ++q) slow = rates[q] < slow ? rates[q] : slow;
  return (double)f / (double)tot * 3.0 / slow;
}

static double sync_cost(int kind, const int64_t *p, const int64_t *o, const int64_t *in, const int64_t *cfg, int nd,
                        const double *bw) { /* :79-94 */
  const double P = param_bytes(kind, p, o, in);
  if (P == 0.0) return 0.0;
  const int64_t tot = cfg_total(cfg);
  if (tot / cfg[1] == 1) return 0.0;
  const double shard = P / (double)cfg[1];
  double t = 0.0;
  for (int64_t q = 1; q < tot; ++q) t += 2.0 * shard / bw[q * nd + 0];
  return t;
}

/* cost.hpp:103-131: per-(p,q) bytes (each pair visited once under identity
 * placement), seconds = max over pairs of bytes/bw, bytes = sum in map order */
static void transfer(const orc_instance *g, int e, const int64_t *cs, const int64_t *cd, int nd, const double *bw,
                     double *sec, double *bytes) {
  const int64_t *sshape = g->shape + 4 * g->esrc[e];
  const int64_t ts = cfg_total(cs), td = cfg_total(cd);
  /* std::map iterates keys (p,q) ascending: collect per pair, then walk p-major */
  double *pb = (double *)xcalloc((size_t)(ts * td), sizeof(double));
  for (int64_t q = 0; q < td; ++q) {
    const region need = required(g, e, cd, q);
    if (reg_volume(&need) == 0) continue;
    for (int64_t p = 0; p < ts; ++p) {
      if (p == q) continue;
      const region o = owned(sshape, cs, p);
      const region x = reg_intersect(&o, &need);
      const int64_t v = reg_volume(&x);
      if (v > 0) pb[p * td + q] += 4.0 * (double)v;
    }
  }
  double s = 0.0, b = 0.0;
  for (int64_t p = 0; p < ts; ++p)
    for (int64_t q = 0; q < td; ++q)
      if (pb[p * td + q] > 0.0) {
        b += pb[p * td + q];
        const double t = pb[p * td + q] / bw[p * nd + q];
        s = t > s ? t : s;
      }
  free(pb);
  *sec = s;
  *bytes = b;
}

int orc_transfer_profile(const orc_instance *g, int e, const int64_t *cs, const int64_t *cd, int nd, const double *bw,
                         double *seconds, double *bytes) {
  if (cfg_total(cs) > nd || cfg_total(cd) > nd) return set_err("config needs more devices than available"), 1;
  transfer(g, e, cs, cd, nd, bw, seconds, bytes);
  return 0;
}

int orc_build_tables(orc_instance *g, int nd, const double *rates, const double *bw) { /* cost.hpp:170-206 */
  if (nd < 1) return set_err("device graph: need at least one device"), 1;
  free_reduced(g);
  free_tables(g);
  g->ncfg = (int *)xcalloc((size_t)g->nl, sizeof(int));
  g->cat = (int64_t **)xcalloc((size_t)g->nl, sizeof(int64_t *));
  g->node = (double **)xcalloc((size_t)g->nl, sizeof(double *));
  g->compute = (double **)xcalloc((size_t)g->nl, sizeof(double *));
  g->sync = (double **)xcalloc((size_t)g->nl, sizeof(double *));
  g->xfer = (double **)xcalloc((size_t)g->ne, sizeof(double *));
  g->have_tables = 1;
  for (int l = 0; l < g->nl; ++l) {
    const int64_t *o = g->shape + 4 * l;
    const int64_t *in = g->in_e[l].n ? g->shape + 4 * g->esrc[g->in_e[l].v[0]] : o; /* :181-182 */
    const int n = orc_enumerate_configs(g->kind[l], o, nd, NULL, 0);
    g->ncfg[l] = n;
    g->cat[l] = (int64_t *)xcalloc((size_t)n * 4, sizeof(int64_t));
    orc_enumerate_configs(g->kind[l], o, nd, g->cat[l], n);
    g->node[l] = (double *)xcalloc((size_t)n, sizeof(double));
    g->compute[l] = (double *)xcalloc((size_t)n, sizeof(double));
    g->sync[l] = (double *)xcalloc((size_t)n, sizeof(double));
    for (int c = 0; c < n; ++c) {
      const double tc = compute_cost(g->kind[l], g->params + 7 * l, o, in, g->cat[l] + 4 * c, rates);
      const double ts = sync_cost(g->kind[l], g->params + 7 * l, o, in, g->cat[l] + 4 * c, nd, bw);
      g->compute[l][c] = tc;
      g->sync[l][c] = ts;
      g->node[l][c] = tc + ts;
    }
  }
  for (int e = 0; e < g->ne; ++e) {
    const int s = g->esrc[e], d = g->edst[e];
    g->xfer[e] = (double *)xcalloc((size_t)g->ncfg[s] * (size_t)g->ncfg[d], sizeof(double));
    for (int i = 0; i < g->ncfg[s]; ++i)
      for (int j = 0; j < g->ncfg[d]; ++j) {
        double sec, by;
        transfer(g, e, g->cat[s] + 4 * i, g->cat[d] + 4 * j, nd, bw, &sec, &by);
        g->xfer[e][(size_t)i * g->ncfg[d] + j] = sec;
      }
  }
  return 0;
}

int orc_set_tables(orc_instance *g, const int32_t *ncfg, const int64_t *configs, const double *node, const double *xfer) {
  free_reduced(g);
  free_tables(g);
  g->ncfg = (int *)xcalloc((size_t)g->nl, sizeof(int));
  g->cat = (int64_t **)xcalloc((size_t)g->nl, sizeof(int64_t *));
  g->node = (double **)xcalloc((size_t)g->nl, sizeof(double *));
  g->compute = (double **)xcalloc((size_t)g->nl, sizeof(double *));
  g->sync = (double **)xcalloc((size_t)g->nl, sizeof(double *));
  g->xfer = (double **)xcalloc((size_t)g->ne, sizeof(double *));
  g->have_tables = 1;
  size_t oc = 0, on = 0, ox = 0;
  for (int l = 0; l < g->nl; ++l) {
    const int n = ncfg[l];
    g->ncfg[l] = n;
    g->cat[l] = (int64_t *)xcalloc((size_t)n * 4, sizeof(int64_t));
    memcpy(g->cat[l], configs + oc, (size_t)n * 4 * sizeof(int64_t));
    oc += (size_t)n * 4;
    g->node[l] = (double *)xcalloc((size_t)n, sizeof(double));
    memcpy(g->node[l], node + on, (size_t)n * sizeof(double));
    on += (size_t)n;
    g->compute[l] = (double *)xcalloc(1, sizeof(double));
    g->sync[l] = (double *)xcalloc(1, sizeof(double));
  }
  for (int e = 0; e < g->ne; ++e) {
    const size_t n = (size_t)ncfg[g->esrc[e]] * (size_t)ncfg[g->edst[e]];
    g->xfer[e] = (double *)xcalloc(n, sizeof(double));
    memcpy(g->xfer[e], xfer + ox, n * sizeof(double));
    ox += n;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* accessors                                                                */
/* ------------------------------------------------------------------------ */

int orc_n_layers(const orc_instance *g) { return g->nl; }
int orc_n_edges(const orc_instance *g) { return g->ne; }
void orc_edges(const orc_instance *g, int32_t *s, int32_t *d, int32_t *p) {
  for (int e = 0; e < g->ne; ++e) {
    if (s) s[e] = g->esrc[e];
    if (d) d[e] = g->edst[e];
    if (p) p[e] = g->epos[e];
  }
}
void orc_shapes(const orc_instance *g, int64_t *o) { memcpy(o, g->shape, (size_t)g->nl * 4 * sizeof(int64_t)); }
void orc_topo(const orc_instance *g, int32_t *o) {
  for (int l = 0; l < g->nl; ++l) o[l] = g->topo[l];
}
int orc_config_count(const orc_instance *g, int l) { return g->have_tables ? g->ncfg[l] : -1; }
void orc_catalog(const orc_instance *g, int l, int64_t *o) { memcpy(o, g->cat[l], (size_t)g->ncfg[l] * 4 * sizeof(int64_t)); }
void orc_node(const orc_instance *g, int l, double *o) { memcpy(o, g->node[l], (size_t)g->ncfg[l] * sizeof(double)); }
void orc_compute(const orc_instance *g, int l, double *o) { memcpy(o, g->compute[l], (size_t)g->ncfg[l] * sizeof(double)); }
void orc_sync(const orc_instance *g, int l, double *o) { memcpy(o, g->sync[l], (size_t)g->ncfg[l] * sizeof(double)); }
void orc_xfer(const orc_instance *g, int e, double *o) {
  memcpy(o, g->xfer[e], (size_t)g->ncfg[g->esrc[e]] * (size_t)g->ncfg[g->edst[e]] * sizeof(double));
}
int orc_layer(const orc_instance *g, int l, int64_t *params, char *id, int cap) {
  if (params) memcpy(params, g->params + 7 * l, 7 * sizeof(int64_t));
  if (id && cap > 0) {
    strncpy(id, g->ids[l], (size_t)cap - 1);
    id[cap - 1] = 0;
  }
  return g->kind[l];
}

/* ------------------------------------------------------------------------ */
/* reduced graph (planner.hpp:55-245)                                       */
/* ------------------------------------------------------------------------ */

static int new_edge(orc_instance *g, int src, int dst, int nu, int nv, double *t) { /* :220-227 */
  if (g->n_redges == g->cap_redges) {
    g->cap_redges = g->cap_redges ? 2 * g->cap_redges : 16;
    g->redges = (orc_redge *)realloc(g->redges, (size_t)g->cap_redges * sizeof(orc_redge));
  }
  const int id = g->n_redges++;
  orc_redge *r = &g->redges[id];
  r->id = id, r->src = src, r->dst = dst, r->alive = 1, r->nu = nu, r->nv = nv, r->t = t;
  iv_push(&g->rin[dst], id);
  iv_push(&g->rout[src], id);
  return id;
}

static void detach(orc_instance *g, int id) { /* :229-236 */
  orc_redge *e = &g->redges[id];
  e->alive = 0;
  iv_erase(&g->rin[e->dst], id);
  iv_erase(&g->rout[e->src], id);
}

static void push_log(orc_instance *g, orc_rec r) {
  if (g->n_log == g->cap_log) {
    g->cap_log = g->cap_log ? 2 * g->cap_log : 16;
    g->log = (orc_rec *)realloc(g->log, (size_t)g->cap_log * sizeof(orc_rec));
  }
  g->log[g->n_log++] = r;
}

static void rg_init(orc_instance *g) { /* :57-69 */
  free_reduced(g);
  g->reduced = 1;
  g->alive = (int *)xcalloc((size_t)g->nl, sizeof(int));
  for (int l = 0; l < g->nl; ++l) g->alive[l] = 1;
  g->rin = (ivec *)xcalloc((size_t)g->nl, sizeof(ivec));
  g->rout = (ivec *)xcalloc((size_t)g->nl, sizeof(ivec));
  for (int e = 0; e < g->ne; ++e) {
    const int nu = g->ncfg[g->esrc[e]], nv = g->ncfg[g->edst[e]];
    double *t = (double *)xcalloc((size_t)nu * (size_t)nv, sizeof(double));
    memcpy(t, g->xfer[e], (size_t)nu * (size_t)nv * sizeof(double));
    new_edge(g, g->esrc[e], g->edst[e], nu, nv, t);
  }
}

void orc_fold(int nu, int nw, int nv, const double *w, const double *t1, const double *t2, double *out, int32_t *am) {
  /* planner.hpp:141-155: (w[j] + t1[i][j]) + t2[j][k], strict < keeps the lowest j */
  for (int i = 0; i < nu; ++i)
    for (int k = 0; k < nv; ++k) {
      double best = w[0] + t1[(size_t)i * nw + 0] + t2[k];
      int bj = 0;
      for (int j = 1; j < nw; ++j) {
        const double c = w[j] + t1[(size_t)i * nw + j] + t2[(size_t)j * nv + k];
        if (c < best) best = c, bj = j;
      }
      out[(size_t)i * nv + k] = best;
      am[(size_t)i * nv + k] = bj;
    }
}

static int node_elimination(orc_instance *g) { /* :114-163 */
  int chosen = -1;
  for (int r = 0; r < g->nl; ++r) {
    const int l = g->topo[r];
    if (g->alive[l] && g->rin[l].n == 1 && g->rout[l].n == 1) {
      chosen = l;
      break;
    }
  }
  if (chosen < 0) return 0;
  const int e1 = g->rin[chosen].v[0], e2 = g->rout[chosen].v[0];
  const int u = g->redges[e1].src, v = g->redges[e2].dst;
  const int nu = g->redges[e1].nu, nw = g->ncfg[chosen], nv = nw ? g->redges[e2].nv : 0;
  double *out = (double *)xcalloc((size_t)nu * (size_t)nv, sizeof(double));
  int32_t *am = (int32_t *)xcalloc((size_t)nu * (size_t)nv, sizeof(int32_t));
  orc_fold(nu, nw, nv, g->node[chosen], g->redges[e1].t, g->redges[e2].t, out, am);
  const int ne = new_edge(g, u, v, nu, nv, out);
  detach(g, e1);
  detach(g, e2);
  g->alive[chosen] = 0;
  orc_rec r = {0, chosen, e1, e2, ne, u, v, nu, nv, am};
  push_log(g, r);
  return 1;
}

static int edge_elimination(orc_instance *g) { /* :167-206 */
  int b1 = -1, b2 = -1;
  for (int a = 0; a < g->n_redges; ++a) {
    const orc_redge *A = &g->redges[a];
    if (!A->alive) continue;
    for (int b = a + 1; b < g->n_redges; ++b) {
      const orc_redge *B = &g->redges[b];
      if (!B->alive || A->src != B->src || A->dst != B->dst) continue;
      int better = b1 < 0;
      if (!better) {
        const orc_redge *X = &g->redges[b1];
        if (A->src != X->src) better = A->src < X->src;
        else if (A->dst != X->dst) better = A->dst < X->dst;
        else if (a != b1) better = a < b1;
        else better = b < b2;
      }
      if (better) b1 = a, b2 = b;
    }
  }
  if (b1 < 0) return 0;
  const orc_redge *A = &g->redges[b1], *B = &g->redges[b2];
  const int u = A->src, v = A->dst, nu = A->nu, nv = A->nv;
  double *sum = (double *)xcalloc((size_t)nu * (size_t)nv, sizeof(double));
  for (size_t k = 0; k < (size_t)nu * (size_t)nv; ++k) sum[k] = A->t[k] + B->t[k];
  const int ne = new_edge(g, u, v, nu, nv, sum);
  detach(g, b1);
  detach(g, b2);
  orc_rec r = {1, -1, b1, b2, ne, u, v, 0, 0, NULL};
  push_log(g, r);
  return 1;
}

int orc_rg_init(orc_instance *g) { /* ReducedGraph ctor (:57-69) */
  if (!g->have_tables) return set_err("no tables"), 1;
  rg_init(g);
  return 0;
}
int orc_rg_node(orc_instance *g) { return g->reduced ? node_elimination(g) : -1; }
int orc_rg_edge(orc_instance *g) { return g->reduced ? edge_elimination(g) : -1; }
int orc_rg_edges_total(const orc_instance *g) { return g->reduced ? g->n_redges : 0; }
int orc_rg_edge_info(const orc_instance *g, int e, int32_t *info3) {
  if (!g->reduced || e < 0 || e >= g->n_redges) return 1;
  info3[0] = g->redges[e].src, info3[1] = g->redges[e].dst, info3[2] = g->redges[e].alive;
  return 0;
}

int orc_reduce(orc_instance *g) { /* :209-217 */
  if (!g->have_tables) return set_err("no tables"), 1;
  rg_init(g);
  for (;;) {
    if (node_elimination(g)) continue;
    if (edge_elimination(g)) continue;
    break;
  }
  return 0;
}

int orc_log_size(const orc_instance *g) { return g->reduced ? g->n_log : 0; }
int orc_log_record(const orc_instance *g, int r, int32_t *o) {
  const orc_rec *x = &g->log[r];
  o[0] = x->type, o[1] = x->removed, o[2] = x->e1, o[3] = x->e2, o[4] = x->ne, o[5] = x->src, o[6] = x->dst;
  return 0;
}
int orc_log_argmin(const orc_instance *g, int r, int32_t *o) {
  const orc_rec *x = &g->log[r];
  if (x->type) return 1;
  memcpy(o, x->argmin, (size_t)x->nu * (size_t)x->nv * sizeof(int32_t));
  return 0;
}
int orc_edge_table_dims(const orc_instance *g, int e, int32_t *d) {
  if (!g->reduced || e < 0 || e >= g->n_redges) return 1;
  d[0] = g->redges[e].nu, d[1] = g->redges[e].nv;
  return 0;
}
int orc_edge_table(const orc_instance *g, int e, double *o) {
  if (!g->reduced || e < 0 || e >= g->n_redges) return 1;
  memcpy(o, g->redges[e].t, (size_t)g->redges[e].nu * (size_t)g->redges[e].nv * sizeof(double));
  return 0;
}
int orc_live_nodes(const orc_instance *g, int32_t *o) {
  int n = 0;
  for (int l = 0; l < g->nl; ++l)
    if (!g->reduced || g->alive[l]) {
      if (o) o[n] = l;
      ++n;
    }
  return n;
}

int orc_enumerate_final(orc_instance *g, int kb, int32_t *idx_out, double *cost_out) { /* :256-304 */
  const int k = orc_live_nodes(g, NULL);
  if (k > kb)
    return set_err("final graph has %d nodes, exceeding the enumeration bound of %d (graph is not reducible enough)", k,
                   kb),
           2;
  int32_t *nodes = (int32_t *)xcalloc((size_t)k, sizeof(int32_t));
  orc_live_nodes(g, nodes);
  int *pos = (int *)xcalloc((size_t)g->nl, sizeof(int));
  for (int l = 0; l < g->nl; ++l) pos[l] = -1;
  for (int i = 0; i < k; ++i) pos[nodes[i]] = i;
  int *idx = (int *)xcalloc((size_t)k, sizeof(int));
  int *best = (int *)xcalloc((size_t)k, sizeof(int));
  double bc = 0.0;
  int have = 0;
  for (;;) {
    double c = 0.0;
    for (int i = 0; i < k; ++i) c += g->node[nodes[i]][idx[i]];
    for (int e = 0; g->reduced && e < g->n_redges; ++e) {
      const orc_redge *r = &g->redges[e];
      if (!r->alive) continue;
      c += r->t[(size_t)idx[pos[r->src]] * r->nv + idx[pos[r->dst]]];
    }
    if (!g->reduced)
      for (int e = 0; e < g->ne; ++e)
        c += g->xfer[e][(size_t)idx[pos[g->esrc[e]]] * g->ncfg[g->edst[e]] + idx[pos[g->edst[e]]]];
    if (!have || c < bc) {
      bc = c;
      memcpy(best, idx, (size_t)k * sizeof(int));
      have = 1;
    }
    int d = k - 1;
    while (d >= 0 && idx[d] + 1 == g->ncfg[nodes[d]]) idx[d--] = 0;
    if (d < 0) break;
    ++idx[d];
  }
  for (int i = 0; i < k; ++i) idx_out[i] = best[i];
  *cost_out = bc;
  free(nodes), free(pos), free(idx), free(best);
  return 0;
}

double orc_total_cost(const orc_instance *g, const int32_t *idx) { /* cost.hpp:235-246 */
  double t = 0.0;
  for (int l = 0; l < g->nl; ++l) t += g->node[l][idx[l]];
  for (int e = 0; e < g->ne; ++e) t += g->xfer[e][(size_t)idx[g->esrc[e]] * g->ncfg[g->edst[e]] + idx[g->edst[e]]];
  return t;
}

int orc_plan(orc_instance *g, int kb, int32_t *indices, double *cost, int32_t *stats) { /* planner.hpp:339-366 */
  if (orc_reduce(g)) return 1;
  const int k = orc_live_nodes(g, NULL);
  int32_t *fin = (int32_t *)xcalloc((size_t)(k ? k : 1), sizeof(int32_t));
  double fc;
  const int st = orc_enumerate_final(g, kb, fin, &fc);
  if (st) return free(fin), st;
  int32_t *nodes = (int32_t *)xcalloc((size_t)(k ? k : 1), sizeof(int32_t));
  orc_live_nodes(g, nodes);
  for (int l = 0; l < g->nl; ++l) indices[l] = -1;
  for (int i = 0; i < k; ++i) indices[nodes[i]] = fin[i];
  int nn = 0, en = 0;
  for (int r = g->n_log - 1; r >= 0; --r) { /* unwind (:309-319) */
    const orc_rec *x = &g->log[r];
    if (x->type) continue;
    indices[x->removed] = x->argmin[(size_t)indices[x->src] * x->nv + indices[x->dst]];
  }
  for (int r = 0; r < g->n_log; ++r) {
    if (g->log[r].type) ++en;
    else ++nn;
  }
  stats[0] = k, stats[1] = nn, stats[2] = en;
  *cost = orc_total_cost(g, indices);
  free(fin), free(nodes);
  return 0;
}

int orc_brute(const orc_instance *g, uint64_t budget, int32_t *indices, double *cost, uint64_t *visited) {
  /* oracle.hpp:52-93 */
  long double space = 1.0L;
  for (int l = 0; l < g->nl; ++l) space *= (long double)g->ncfg[l];
  if (space > (long double)budget) {
    if (space < 1e15L)
      set_err("strategy space has %llu strategies, exceeding the exhaustive-search budget of %llu",
              (unsigned long long)space, (unsigned long long)budget);
    else
      set_err("strategy space has %g strategies, exceeding the exhaustive-search budget of %llu", (double)space,
              (unsigned long long)budget);
    return 2;
  }
  int32_t *idx = (int32_t *)xcalloc((size_t)g->nl, sizeof(int32_t));
  uint64_t vis = 0;
  double bc = 0.0;
  int have = 0;
  for (;;) {
    ++vis;
    const double c = orc_total_cost(g, idx);
    if (!have || c < bc) {
      bc = c;
      memcpy(indices, idx, (size_t)g->nl * sizeof(int32_t));
      have = 1;
    }
    int d = g->nl - 1;
    while (d >= 0 && idx[d] + 1 == g->ncfg[d]) idx[d--] = 0;
    if (d < 0) break;
    ++idx[d];
  }
  free(idx);
  *cost = bc;
  *visited = vis;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* seeded instances (oracle.hpp:121-185; SURVEY §9 config-5 variant)        */
/* ------------------------------------------------------------------------ */

static orc_instance *sp_topology(mt64 *m, int node_count, double bp) { /* oracle.hpp:130-157 */
  builder b;
  memset(&b, 0, sizeof b);
  char id[32];
  int64_t inp[7] = {4, 1, 1, 0, 0, 0, 0}, cat[7] = {1, 0, 0, 0, 0, 0, 0};
#define NID() (snprintf(id, sizeof id, "n%d", b.nl), id)
  int tip = b_add(&b, NID(), ORC_INPUT, inp, 0, NULL);
  int count = 1;
  while (count < node_count) {
    int branch = 0;
    if (node_count - count >= 3) branch = (double)(mt_next(m) % 1000) / 1000.0 < bp;
    if (branch) {
      int a = b_add(&b, NID(), ORC_SOFTMAX, NULL, 1, &tip);
      int c = b_add(&b, NID(), ORC_SOFTMAX, NULL, 1, &tip);
      int ins[2] = {a, c};
      tip = b_add(&b, NID(), ORC_CONCAT, cat, 2, ins);
      count += 3;
    } else {
      tip = b_add(&b, NID(), ORC_SOFTMAX, NULL, 1, &tip);
      count += 1;
    }
  }
#undef NID
  return b_build(&b, 8);
}

static double dyadic(mt64 *m) { return (double)(mt_next(m) % 641) / 64.0; }

orc_instance *orc_random(uint64_t seed, int n, int maxc, double bp, int ndev) {
  g_err[0] = 0;
  if (n < 1) return set_err("random graph needs at least one node"), NULL;
  if (maxc < 1) return set_err("random graph needs at least one config per layer"), NULL;
  if (ndev < 1) return set_err("random graph needs at least one device"), NULL;
  mt64 m;
  mt_seed(&m, seed);
  orc_instance *g = sp_topology(&m, n, bp);
  if (!g) return NULL;
  int32_t *ncfg = (int32_t *)xcalloc((size_t)g->nl, sizeof(int32_t));
  int64_t *cfgs = (int64_t *)xcalloc((size_t)g->nl * 4 * (size_t)maxc, sizeof(int64_t));
  size_t tot = 0, tx = 0;
  for (int l = 0; l < g->nl; ++l) { /* oracle.hpp:164-173: truncate the catalog */
    int64_t tmp[4 * 512];
    int c = orc_enumerate_configs(g->kind[l], g->shape + 4 * l, ndev, tmp, 512);
    if (c > maxc) c = maxc;
    ncfg[l] = c;
    memcpy(cfgs + 4 * tot, tmp, (size_t)c * 4 * sizeof(int64_t));
    tot += (size_t)c;
  }
  for (int e = 0; e < g->ne; ++e) tx += (size_t)ncfg[g->esrc[e]] * (size_t)ncfg[g->edst[e]];
  double *node = (double *)xcalloc(tot, sizeof(double));
  double *xf = (double *)xcalloc(tx, sizeof(double));
  for (size_t k = 0; k < tot; ++k) node[k] = dyadic(&m); /* layers by index */
  for (size_t k = 0; k < tx; ++k) xf[k] = dyadic(&m);    /* edges by id, row-major */
  orc_set_tables(g, ncfg, cfgs, node, xf);
  free(ncfg), free(cfgs), free(node), free(xf);
  return g;
}

orc_instance *orc_synthetic(uint64_t seed, int n, int C, double bp) {
  g_err[0] = 0;
  if (n < 1 || C < 1) return set_err("synthetic graph needs nodes and configs"), NULL;
  mt64 m;
  mt_seed(&m, seed);
  orc_instance *g = sp_topology(&m, n, bp);
  if (!g) return NULL;
  int32_t *ncfg = (int32_t *)xcalloc((size_t)g->nl, sizeof(int32_t));
  int64_t *cfgs = (int64_t *)xcalloc((size_t)g->nl * 4 * (size_t)C, sizeof(int64_t));
  for (int l = 0; l < g->nl; ++l) {
    ncfg[l] = C;
    for (int i = 0; i < C; ++i) {
      int64_t *c = cfgs + 4 * ((size_t)l * C + i);
      c[0] = 1, c[1] = 1, c[2] = 1, c[3] = i + 1;
    }
  }
  const size_t tot = (size_t)g->nl * C, tx = (size_t)g->ne * C * C;
  double *node = (double *)xcalloc(tot, sizeof(double));
  double *xf = (double *)xcalloc(tx, sizeof(double));
  for (size_t k = 0; k < tot; ++k) node[k] = dyadic(&m);
  for (size_t k = 0; k < tx; ++k) xf[k] = dyadic(&m);
  orc_set_tables(g, ncfg, cfgs, node, xf);
  free(ncfg), free(cfgs), free(node), free(xf);
  return g;
}
