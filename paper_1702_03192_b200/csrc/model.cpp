// GBDT selector model in host C++: JSON v1 reader, packed-tree walkers and the
// Algorithm 2 decision.
//
// Reference: model document gbdt.py:388-455 (serialize/deserialize, error
// messages with JSON-path locations), prediction gbdt.py:242-259 (raw >= 0 => +1,
// i.e. NT), packing selector.py:82-123, walkers _numba_impl.py:197-222, decision
// selector.py:181-190. Compiled with -ffp-contract=off so `raw += eta * leaf` is
// the same two roundings as the reference's float64 Python/numba arithmetic, and
// numbers are parsed with strtod (correctly rounded), so Python-repr floats
// round-trip bit-exactly and the label equals gbdt.predict on the same model.
#include "model.h"

#include <errno.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <memory>
#include <chrono>
#include <string>
#include <vector>

#include "common.h"

namespace mtnn {

double walk_packed(const int64_t* feat, const double* thresh, const int64_t* left,
                   const int64_t* right, const double* leaf, int64_t n_trees, int64_t width,
                   const double* x, double base_score, double eta) {
  double raw = base_score;
  for (int64_t t = 0; t < n_trees; ++t) {
    const int64_t off = t * width;
    int64_t node = 0;
    while (feat[off + node] >= 0) {
      node = (x[feat[off + node]] < thresh[off + node]) ? left[off + node] : right[off + node];
    }
    raw += eta * leaf[off + node];
  }
  return raw;
}

namespace {

// ------------------------------------------------------------- tiny JSON DOM
struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  bool is_int = false;  // number literal without fraction/exponent
  double num = 0.0;
  long long inum = 0;
  std::string str;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const char* key) const {
    for (auto& kv : obj)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
};

struct Parser {
  const char* p;
  const char* end;
  std::string err;
  int depth = 0;

  void ws() {
    while (p < end && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  bool fail_at(const char* what) {
    if (err.empty()) err = what;
    return false;
  }
  bool lit(const char* s) {
    size_t n = strlen(s);
    if ((size_t)(end - p) >= n && memcmp(p, s, n) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  bool parse_string(std::string& out) {
    if (p >= end || *p != '"') return fail_at("expected string");
    ++p;
    while (p < end && *p != '"') {
      if (*p == '\\') {
        ++p;
        if (p >= end) return fail_at("bad escape");
        switch (*p) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {
            if (end - p < 5) return fail_at("bad unicode escape");
            unsigned cp = (unsigned)strtoul(std::string(p + 1, p + 5).c_str(), nullptr, 16);
            if (cp < 0x80) out += (char)cp; else out += '?';
            p += 4;
            break;
          }
          default: return fail_at("bad escape");
        }
        ++p;
      } else {
        out += *p++;
      }
    }
    if (p >= end) return fail_at("unterminated string");
    ++p;
    return true;
  }
  bool parse_number(JVal& v) {
    const char* s = p;
    bool frac = false;
    if (p < end && *p == '-') ++p;
    if (lit("Infinity")) {
      v.kind = JVal::Num;
      v.num = (*s == '-') ? -INFINITY : INFINITY;
      return true;
    }
    while (p < end && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E' ||
                       *p == '+' || *p == '-')) {
      if (*p == '.' || *p == 'e' || *p == 'E') frac = true;
      ++p;
    }
    if (p == s) return fail_at("expected value");
    std::string tok(s, p);
    char* ep = nullptr;
    errno = 0;
    v.kind = JVal::Num;
    v.num = strtod(tok.c_str(), &ep);
    if (ep == nullptr || *ep != '\0') return fail_at("bad number");
    v.is_int = !frac;
    if (v.is_int) v.inum = strtoll(tok.c_str(), nullptr, 10);
    return true;
  }
  bool parse(JVal& v) {
    if (++depth > 512) return fail_at("nesting too deep");
    ws();
    if (p >= end) return fail_at("unexpected end of input");
    bool ok = true;
    if (*p == '{') {
      ++p;
      v.kind = JVal::Obj;
      ws();
      if (p < end && *p == '}') { ++p; --depth; return true; }
      while (true) {
        ws();
        std::string key;
        if (!parse_string(key)) return false;
        ws();
        if (p >= end || *p != ':') return fail_at("expected ':'");
        ++p;
        JVal child;
        if (!parse(child)) return false;
        // duplicate keys: last one wins (Python json semantics)
        bool replaced = false;
        for (auto& kv : v.obj)
          if (kv.first == key) { kv.second = std::move(child); replaced = true; break; }
        if (!replaced) v.obj.emplace_back(std::move(key), std::move(child));
        ws();
        if (p < end && *p == ',') { ++p; continue; }
        if (p < end && *p == '}') { ++p; break; }
        return fail_at("expected ',' or '}'");
      }
    } else if (*p == '[') {
      ++p;
      v.kind = JVal::Arr;
      ws();
      if (p < end && *p == ']') { ++p; --depth; return true; }
      while (true) {
        JVal child;
        if (!parse(child)) return false;
        v.arr.push_back(std::move(child));
        ws();
        if (p < end && *p == ',') { ++p; continue; }
        if (p < end && *p == ']') { ++p; break; }
        return fail_at("expected ',' or ']'");
      }
    } else if (*p == '"') {
      v.kind = JVal::Str;
      ok = parse_string(v.str);
    } else if (lit("true")) {
      v.kind = JVal::Bool; v.b = true;
    } else if (lit("false")) {
      v.kind = JVal::Bool; v.b = false;
    } else if (lit("null")) {
      v.kind = JVal::Null;
    } else if (lit("NaN")) {
      v.kind = JVal::Num; v.num = NAN;
    } else {
      ok = parse_number(v);
    }
    --depth;
    return ok;
  }
};

struct Node {
  bool is_leaf = true;
  int64_t feature = -1;
  double threshold = 0.0, weight = 0.0;
  std::unique_ptr<Node> left, right;
};

int node_from(const JVal& v, const std::string& where, std::unique_ptr<Node>& out) {
  if (v.kind != JVal::Obj)
    return fail(MTNN_EINVAL, "%s: expected an object", where.c_str());
  auto n = std::make_unique<Node>();
  if (const JVal* lf = v.get("leaf")) {
    if (lf->kind != JVal::Num) return fail(MTNN_EINVAL, "%s.leaf: expected a number", where.c_str());
    n->is_leaf = true;
    n->weight = lf->num;
    out = std::move(n);
    return MTNN_OK;
  }
  for (const char* key : {"feat", "thresh", "left", "right"})
    if (!v.get(key)) return fail(MTNN_EINVAL, "%s: missing '%s'", where.c_str(), key);
  const JVal* f = v.get("feat");
  if (f->kind != JVal::Num || !f->is_int || f->inum < 0)
    return fail(MTNN_EINVAL, "%s.feat: expected a non-negative integer", where.c_str());
  const JVal* t = v.get("thresh");
  if (t->kind != JVal::Num) return fail(MTNN_EINVAL, "%s.thresh: expected a number", where.c_str());
  n->is_leaf = false;
  n->feature = f->inum;
  n->threshold = t->num;
  MTNN_TRY(node_from(*v.get("left"), where + ".left", n->left));
  MTNN_TRY(node_from(*v.get("right"), where + ".right", n->right));
  out = std::move(n);
  return MTNN_OK;
}

int64_t count_nodes(const Node* n) {
  return n->is_leaf ? 1 : 1 + count_nodes(n->left.get()) + count_nodes(n->right.get());
}

int64_t place(const Node* n, mtnn_model* m, int64_t t, int64_t& next) {
  const int64_t idx = next++;
  const int64_t o = t * m->width + idx;
  if (n->is_leaf) {
    m->leaf[o] = n->weight;
    return idx;
  }
  m->feat[o] = n->feature;
  m->thresh[o] = n->threshold;
  m->left[o] = place(n->left.get(), m, t, next);
  m->right[o] = place(n->right.get(), m, t, next);
  return idx;
}

double num_of(const JVal* v, bool* ok) {
  if (!v) { *ok = false; return 0.0; }
  if (v->kind == JVal::Num) return v->num;
  if (v->kind == JVal::Bool) return v->b ? 1.0 : 0.0;
  if (v->kind == JVal::Str) {
    char* ep = nullptr;
    double d = strtod(v->str.c_str(), &ep);
    if (ep && *ep == '\0' && !v->str.empty()) return d;
  }
  *ok = false;
  return 0.0;
}

}  // namespace

int model_from_trees(std::vector<std::unique_ptr<Node>>& trees, double base, double eta,
                     int64_t n_features, mtnn_model** out) {
  auto m = std::make_unique<mtnn_model>();
  m->n_trees = trees.empty() ? 1 : (int64_t)trees.size();
  int64_t width = 1;
  for (auto& t : trees) width = std::max<int64_t>(width, count_nodes(t.get()));
  m->width = width;
  m->base_score = base;
  m->eta = eta;
  m->n_features = n_features;
  const size_t cells = (size_t)(m->n_trees * width);
  for (auto& t : trees) {
    int64_t mf = -1;
    std::vector<const Node*> st{t.get()};
    while (!st.empty()) {
      const Node* nd = st.back();
      st.pop_back();
      if (!nd->is_leaf) {
        mf = std::max(mf, nd->feature);
        st.push_back(nd->left.get());
        st.push_back(nd->right.get());
      }
    }
    if (mf >= n_features)
      return fail(MTNN_EINVAL, "$.trees: feature index %lld out of range for n_features=%lld",
                  (long long)mf, (long long)n_features);
  }
  m->feat.assign(cells, -1);
  m->thresh.assign(cells, 0.0);
  m->left.assign(cells, 0);
  m->right.assign(cells, 0);
  m->leaf.assign(cells, 0.0);
  for (size_t t = 0; t < trees.size(); ++t) {
    int64_t next = 0;
    place(trees[t].get(), m.get(), (int64_t)t, next);
  }
  *out = m.release();
  return MTNN_OK;
}

}  // namespace mtnn

using namespace mtnn;

extern "C" {

double mtnn_walk_trees(const int64_t* feat, const double* thresh, const int64_t* left,
                       const int64_t* right, const double* leaf, int64_t n_trees,
                       int64_t width, const double* x, double base_score, double eta) {
  return walk_packed(feat, thresh, left, right, leaf, n_trees, width, x, base_score, eta);
}

double mtnn_walk_trees_mnk(const int64_t* feat, const double* thresh, const int64_t* left,
                           const int64_t* right, const double* leaf, int64_t n_trees,
                           int64_t width, const double* prefix5, double m, double n,
                           double k, double base_score, double eta) {
  const double x[8] = {prefix5[0], prefix5[1], prefix5[2], prefix5[3], prefix5[4], m, n, k};
  return walk_packed(feat, thresh, left, right, leaf, n_trees, width, x, base_score, eta);
}

int mtnn_model_load_json(const char* text, size_t len, mtnn_model** out) {
  if (!text || !out) return fail(MTNN_EINVAL, "null argument");
  Parser ps{text, text + len, {}};
  JVal doc;
  if (!ps.parse(doc)) return fail(MTNN_EINVAL, "not valid JSON: %s", ps.err.c_str());
  ps.ws();
  if (ps.p != ps.end) return fail(MTNN_EINVAL, "not valid JSON: extra data");
  if (doc.kind != JVal::Obj) return fail(MTNN_EINVAL, "$: expected a JSON object");
  for (const char* key : {"version", "params", "base_score", "trees"})
    if (!doc.get(key)) return fail(MTNN_EINVAL, "$: missing '%s'", key);
  const JVal* ver = doc.get("version");
  if (!(ver->kind == JVal::Num && ver->num == 1.0))
    return fail(MTNN_EINVAL, "$.version: unsupported version");
  const JVal* params = doc.get("params");
  if (params->kind != JVal::Obj) return fail(MTNN_EINVAL, "$.params: expected an object");
  for (const char* key : {"max_depth", "n_estimators", "eta", "gamma", "lambda", "min_child_weight"})
    if (!params->get(key)) return fail(MTNN_EINVAL, "$.params: missing '%s'", key);
  bool ok = true;
  const double max_depth = num_of(params->get("max_depth"), &ok);
  const double n_est = num_of(params->get("n_estimators"), &ok);
  const double eta = num_of(params->get("eta"), &ok);
  (void)num_of(params->get("gamma"), &ok);
  (void)num_of(params->get("lambda"), &ok);
  (void)num_of(params->get("min_child_weight"), &ok);
  if (!ok) return fail(MTNN_EINVAL, "$.params: non-numeric parameter");
  if ((int64_t)max_depth < 1) return fail(MTNN_EINVAL, "$.params: max_depth must be >= 1");
  if ((int64_t)n_est < 1) return fail(MTNN_EINVAL, "$.params: n_estimators must be >= 1");
  if (const JVal* obj = params->get("objective")) {
    if (obj->kind != JVal::Str || (obj->str != "logistic" && obj->str != "squared"))
      return fail(MTNN_EINVAL, "$.params: unknown objective");
  }
  const JVal* trees = doc.get("trees");
  if (trees->kind != JVal::Arr) return fail(MTNN_EINVAL, "$.trees: expected a list");
  std::vector<std::unique_ptr<Node>> nodes;
  for (size_t i = 0; i < trees->arr.size(); ++i) {
    std::unique_ptr<Node> n;
    MTNN_TRY(node_from(trees->arr[i], "$.trees[" + std::to_string(i) + "]", n));
    nodes.push_back(std::move(n));
  }
  if ((int64_t)nodes.size() > (int64_t)n_est)
    return fail(MTNN_EINVAL, "$.trees: %zu trees exceeds n_estimators=%lld", nodes.size(),
                (long long)n_est);
  bool bok = true;
  const double base = num_of(doc.get("base_score"), &bok);
  if (!bok) return fail(MTNN_EINVAL, "$.base_score: expected a number");
  int64_t n_features = 8;
  if (const JVal* nf = doc.get("n_features")) {
    bool nok = true;
    n_features = (int64_t)num_of(nf, &nok);
    if (!nok) return fail(MTNN_EINVAL, "$.n_features: expected a number");
  }
  return model_from_trees(nodes, base, eta, n_features, out);
}

int mtnn_model_from_packed(const int64_t* feat, const double* thresh, const int64_t* left,
                           const int64_t* right, const double* leaf, int64_t n_trees,
                           int64_t width, double base_score, double eta, int64_t n_features,
                           mtnn_model** out) {
  if (!out || !feat || !thresh || !left || !right || !leaf)
    return fail(MTNN_EINVAL, "null argument");
  if (n_trees < 1 || width < 1) return fail(MTNN_EINVAL, "packed model must have >= 1 tree and node");
  const size_t cells = (size_t)(n_trees * width);
  // structural check so a walk can never leave the arrays
  for (size_t i = 0; i < cells; ++i) {
    if (feat[i] >= 0) {
      if (feat[i] >= n_features)
        return fail(MTNN_EINVAL, "packed node %zu uses feature %lld >= %lld", i,
                    (long long)feat[i], (long long)n_features);
      if (left[i] < 0 || left[i] >= width || right[i] < 0 || right[i] >= width)
        return fail(MTNN_EINVAL, "packed node %zu has out-of-range children", i);
    }
  }
  auto m = std::make_unique<mtnn_model>();
  m->n_trees = n_trees;
  m->width = width;
  m->base_score = base_score;
  m->eta = eta;
  m->n_features = n_features;
  m->feat.assign(feat, feat + cells);
  m->thresh.assign(thresh, thresh + cells);
  m->left.assign(left, left + cells);
  m->right.assign(right, right + cells);
  m->leaf.assign(leaf, leaf + cells);
  *out = m.release();
  return MTNN_OK;
}

void mtnn_model_free(mtnn_model* model) { delete model; }

int64_t mtnn_model_n_features(const mtnn_model* model) { return model ? model->n_features : -1; }
int64_t mtnn_model_n_trees(const mtnn_model* model) { return model ? model->n_trees : -1; }

int mtnn_model_raw(const mtnn_model* model, const double* x, int64_t nx, double* raw) {
  if (!model || !x || !raw) return fail(MTNN_EINVAL, "null argument");
  if (nx != model->n_features)
    return fail(MTNN_EINVAL, "expected %lld features, got shape (%lld,)",
                (long long)model->n_features, (long long)nx);
  for (int64_t i = 0; i < nx; ++i)
    if (!isfinite(x[i])) return fail(MTNN_EINVAL, "features must be finite");
  for (size_t i = 0; i < model->feat.size(); ++i)
    if (model->feat[i] >= nx)
      return fail(MTNN_EINVAL, "model uses feature %lld but only %lld given",
                  (long long)model->feat[i], (long long)nx);
  *raw = walk_packed(model->feat.data(), model->thresh.data(), model->left.data(),
                     model->right.data(), model->leaf.data(), model->n_trees, model->width, x,
                     model->base_score, model->eta);
  return MTNN_OK;
}

int mtnn_select(const mtnn_model* model, const double prefix5[5], int64_t m, int64_t n,
                int64_t k, int64_t free_bytes, double* raw_out, int* choice_out,
                int* reason_out) {
  if (!model || !prefix5) return fail(MTNN_EINVAL, "null argument");
  if (model->n_features != 8)
    return fail(MTNN_EINVAL, "dispatch model must take 8 features, got %lld",
                (long long)model->n_features);
  if (free_bytes < 0) MTNN_TRY(mtnn_device_free_bytes(&free_bytes));
  double raw;
  int choice, reason;
  if (4.0 * (double)n * (double)k > (double)free_bytes) {
    raw = NAN;
    choice = MTNN_CHOICE_NT;
    reason = MTNN_REASON_MEMORY_FALLBACK;
  } else {
    const double x[8] = {prefix5[0], prefix5[1], prefix5[2], prefix5[3], prefix5[4],
                         (double)m, (double)n, (double)k};
    raw = walk_packed(model->feat.data(), model->thresh.data(), model->left.data(),
                      model->right.data(), model->leaf.data(), model->n_trees, model->width, x,
                      model->base_score, model->eta);
    choice = raw >= 0.0 ? MTNN_CHOICE_NT : MTNN_CHOICE_TNN;
    reason = MTNN_REASON_PREDICTED;
  }
  if (raw_out) *raw_out = raw;
  if (choice_out) *choice_out = choice;
  if (reason_out) *reason_out = reason;
  return MTNN_OK;
}

int mtnn_select_cost_ns(const mtnn_model* model, const double prefix5[5], int64_t iters,
                        double* ns_per_call) {
  if (!model || !prefix5 || !ns_per_call || iters <= 0) return fail(MTNN_EINVAL, "bad argument");
  // shapes from the sweep grid, cycled, so the walk takes different branches
  static const int64_t dims[8] = {128, 256, 512, 1024, 2048, 4096, 8192, 16384};
  volatile int sink = 0;
  const auto t0 = std::chrono::steady_clock::now();
  for (int64_t i = 0; i < iters; ++i) {
    double raw;
    int choice, reason;
    const int rc = mtnn_select(model, prefix5, dims[i & 7], dims[(i >> 3) & 7], dims[(i >> 6) & 7],
                               int64_t(1) << 40, &raw, &choice, &reason);
    if (rc != MTNN_OK) return rc;
    sink = sink + choice;
  }
  const auto t1 = std::chrono::steady_clock::now();
  (void)sink;
  *ns_per_call = std::chrono::duration<double, std::nano>(t1 - t0).count() / (double)iters;
  return MTNN_OK;
}

}  // extern "C"
