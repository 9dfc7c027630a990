// qpk_multi.cuh -- one process driving several GPUs (included by qpk.cu).  The reference's solve() is a single process (ipm.py:185-206);
// this layer lets its unmodified direction_solver hook use N GPUs: one
// qpk_ctx per device, each holding a contiguous nnz-balanced row shard of B,
// one host thread per device for every call, the per-iteration all-reduces
// through one NCCL communicator per device (ncclCommInitRank from the N
// threads with one id).  The per-device code path is exactly the sharded
// engine the one-process-per-GPU launcher uses (qpk_shard_init).

struct qpk_multi {
  std::vector<int> devs;
  std::vector<qpk_ctx*> ctx;
  bool comm_ready = false;
  HostComm* hostcomm = nullptr;         // emulated ranks (test only): host-mediated all-reduce
  // problem being described (the caller's arrays stay valid until finalize)
  struct Seg { int64_t n_rows; const int64_t* ro; const int64_t* ci; const double* v; std::vector<int64_t> rows; double sign; };
  std::vector<Seg> segs;
  int64_t n = 0, m_e = 0, m_l = 0, m_u = 0, m = 0;
  int hkind = -1;
  const void* hp[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t hk = 0;
  std::vector<int64_t> lo, hi;          // row bounds of B per device
  bool finalized = false;
  std::vector<std::vector<double>> buf;  // per-device staging of local vectors
};

namespace {

// run fn(r) on one host thread per device; the first failure's message is
// re-raised on the calling thread
template <typename F>
int multi_run(qpk_multi* mm, F fn) {
  const int nd = (int)mm->ctx.size();
  std::vector<int> rc(nd, QPK_OK);
  std::vector<std::string> msg(nd);
  if (nd == 1) {
    rc[0] = fn(0);
    return rc[0];
  }
  std::vector<std::thread> th;
  for (int r = 0; r < nd; ++r)
    th.emplace_back([&, r] {
      rc[r] = fn(r);
      if (rc[r] != QPK_OK) msg[r] = g_err;
    });
  for (auto& t : th) t.join();
  for (int r = 0; r < nd; ++r)
    if (rc[r] != QPK_OK) return fail(rc[r], "device %d: %s", mm->devs[r], msg[r].c_str());
  return QPK_OK;
}

}  // namespace

extern "C" {

int qpk_multi_create(int n_devices, const int* device_ids, qpk_multi** out) {
  if (!out || n_devices < 1 || !device_ids) return fail(QPK_E_ARG, "qpk_multi_create: bad arguments");
  for (int a = 0; a < n_devices; ++a)
    for (int b = a + 1; b < n_devices; ++b)
      if (device_ids[a] == device_ids[b]) return fail(QPK_E_ARG, "qpk_multi_create: device %d listed twice", device_ids[a]);
  qpk_multi* mm = new qpk_multi();
  for (int r = 0; r < n_devices; ++r) {
    qpk_ctx* c = nullptr;
    const int rc = qpk_create(device_ids[r], &c);
    if (rc != QPK_OK) {
      for (qpk_ctx* p : mm->ctx) qpk_destroy(p);
      delete mm;
      return rc;
    }
    mm->devs.push_back(device_ids[r]);
    mm->ctx.push_back(c);
  }
  mm->buf.resize(n_devices);
  *out = mm;
  return QPK_OK;
}

int qpk_multi_destroy(qpk_multi* mm) {
  if (!mm) return QPK_OK;
  for (qpk_ctx* c : mm->ctx) qpk_destroy(c);
  delete mm->hostcomm;
  delete mm;
  return QPK_OK;
}

// Test hook: `n_ranks` contexts on ONE device, their collectives mediated by
// the host (HostComm).  The whole N > 1 sharded engine -- row shards, slices
// of the top block and of the Hessian rows, every all-reduce of a slot, the
// decision kernel -- runs on a single GPU, rank kernels never waiting on one
// another.
int qpk_multi_create_emulated(int n_ranks, int device, qpk_multi** out) {
  if (!out || n_ranks < 1) return fail(QPK_E_ARG, "qpk_multi_create_emulated: bad arguments");
  qpk_multi* mm = new qpk_multi();
  for (int r = 0; r < n_ranks; ++r) {
    qpk_ctx* c = nullptr;
    const int rc = qpk_create(device, &c);
    if (rc != QPK_OK) {
      for (qpk_ctx* p : mm->ctx) qpk_destroy(p);
      delete mm;
      return rc;
    }
    mm->devs.push_back(device);
    mm->ctx.push_back(c);
  }
  mm->buf.resize(n_ranks);
  mm->hostcomm = new HostComm();
  mm->hostcomm->n = n_ranks;
  mm->hostcomm->bufs.resize(n_ranks);
  *out = mm;
  return QPK_OK;
}

int qpk_multi_devices(qpk_multi* mm) { return mm ? (int)mm->ctx.size() : 0; }
qpk_ctx* qpk_multi_context(qpk_multi* mm, int r) { return (mm && r >= 0 && r < (int)mm->ctx.size()) ? mm->ctx[r] : nullptr; }

int qpk_multi_problem_begin(qpk_multi* mm, int64_t n, int64_t m_e, int64_t m_l, int64_t m_u) {
  if (!mm) return fail(QPK_E_ARG, "null context");
  if (n < 1 || m_e < 0 || m_l < 0 || m_u < 0) return fail(QPK_E_ARG, "qpk_multi_problem_begin: bad sizes");
  mm->n = n; mm->m_e = m_e; mm->m_l = m_l; mm->m_u = m_u; mm->m = 0;
  mm->segs.clear();
  mm->hkind = -1;
  mm->finalized = false;
  return QPK_OK;
}

// same arguments as qpk_problem_add_rows; the arrays are read at finalize
int qpk_multi_problem_add_rows(qpk_multi* mm, int64_t n_rows, const int64_t* ro, const int64_t* ci, const double* vals,
                               const int64_t* rows, int64_t n_sel, double sign) {
  if (!mm) return fail(QPK_E_ARG, "null context");
  if (n_rows < 0 || !ro) return fail(QPK_E_ARG, "qpk_multi_problem_add_rows: bad CSR");
  qpk_multi::Seg sg{n_rows, ro, ci, vals, {}, sign};
  const int64_t count = rows ? n_sel : n_rows;
  sg.rows.resize(count);
  for (int64_t s = 0; s < count; ++s) {
    const int64_t i = rows ? rows[s] : s;
    if (i < 0 || i >= n_rows) return fail(QPK_E_ARG, "qpk_multi_problem_add_rows: row index %lld out of range", (long long)i);
    sg.rows[s] = i;
  }
  if (mm->m + count > mm->m_e + mm->m_l + mm->m_u) return fail(QPK_E_ARG, "qpk_multi_problem_add_rows: more rows than m_B");
  mm->m += count;
  mm->segs.push_back(std::move(sg));
  return QPK_OK;
}

int qpk_multi_set_hessian_diag(qpk_multi* mm, const double* d) {
  if (!mm || !d) return fail(QPK_E_ARG, "qpk_multi_set_hessian_diag: bad argument");
  mm->hkind = QPK_HESS_DIAG; mm->hp[0] = d;
  return QPK_OK;
}
int qpk_multi_set_hessian_csr(qpk_multi* mm, const int64_t* ro, const int64_t* ci, const double* v) {
  if (!mm || !ro) return fail(QPK_E_ARG, "qpk_multi_set_hessian_csr: bad argument");
  mm->hkind = QPK_HESS_CSR; mm->hp[0] = ro; mm->hp[1] = ci; mm->hp[2] = v;
  return QPK_OK;
}
int qpk_multi_set_hessian_dense(qpk_multi* mm, const double* m_rowmajor) {
  if (!mm || !m_rowmajor) return fail(QPK_E_ARG, "qpk_multi_set_hessian_dense: bad argument");
  mm->hkind = QPK_HESS_DENSE; mm->hp[0] = m_rowmajor;
  return QPK_OK;
}
int qpk_multi_set_hessian_lowrank(qpk_multi* mm, const double* h0, int64_t k, const double* u, const double* w) {
  if (!mm || !h0) return fail(QPK_E_ARG, "qpk_multi_set_hessian_lowrank: bad argument");
  mm->hkind = QPK_HESS_LOWRANK; mm->hp[0] = h0; mm->hp[1] = u; mm->hp[2] = w; mm->hk = k;
  return QPK_OK;
}

int qpk_multi_problem_finalize(qpk_multi* mm, int scatter) {
  if (!mm) return fail(QPK_E_ARG, "null context");
  if (mm->hkind < 0) return fail(QPK_E_STATE, "qpk_multi_problem_finalize: Hessian not set");
  if (mm->m != mm->m_e + mm->m_l + mm->m_u) return fail(QPK_E_STATE, "qpk_multi_problem_finalize: rows missing");
  const int nd = (int)mm->ctx.size();
  // contiguous row blocks with balanced work (nnz + 1 per row), as sharded.partition_rows
  std::vector<long long> pre(mm->m + 1, 0);
  {
    int64_t g = 0;
    for (const auto& sg : mm->segs)
      for (int64_t i : sg.rows) { pre[g + 1] = pre[g] + (sg.ro[i + 1] - sg.ro[i]) + 1; ++g; }
  }
  mm->lo.assign(nd, 0); mm->hi.assign(nd, 0);
  for (int r = 0; r < nd; ++r) {
    mm->lo[r] = r == 0 ? 0 : (int64_t)(std::lower_bound(pre.begin(), pre.end(), pre.back() * r / nd) - pre.begin());
    mm->hi[r] = r == nd - 1 ? mm->m : (int64_t)(std::lower_bound(pre.begin(), pre.end(), pre.back() * (r + 1) / nd) - pre.begin());
  }
  for (int r = 0; r < nd; ++r) { mm->lo[r] = std::min(mm->lo[r], mm->m); mm->hi[r] = std::max(mm->lo[r], std::min(mm->hi[r], mm->m)); }
  for (int r = 1; r < nd; ++r) mm->lo[r] = mm->hi[r - 1];
  mm->hi[nd - 1] = mm->m;
  // one communicator per device, created from the device threads with one id
  unsigned char id[128];
  if (!mm->comm_ready && !mm->hostcomm) {
    int rc = qpk_nccl_get_unique_id(id);
    if (rc != QPK_OK) return rc;
  }
  int rc = multi_run(mm, [&](int r) -> int {
    qpk_ctx* c = mm->ctx[r];
    if (!mm->comm_ready) {
      if (mm->hostcomm) {                              // emulated ranks: no NCCL
        c->world = nd; c->rank = r; c->sharded = true; c->hostcomm = mm->hostcomm;
      } else {
        int e = qpk_shard_init(c, nd, r, id);
        if (e != QPK_OK) return e;
      }
    }
    int e = qpk_problem_begin(c, mm->n, 0, mm->hi[r] - mm->lo[r], 0);
    if (e != QPK_OK) return e;
    int64_t base = 0;
    for (const auto& sg : mm->segs) {
      const int64_t cnt = (int64_t)sg.rows.size();
      const int64_t a = std::max(mm->lo[r], base), b = std::min(mm->hi[r], base + cnt);
      if (a < b) {
        e = qpk_problem_add_rows(c, sg.n_rows, sg.ro, sg.ci, sg.v, sg.rows.data() + (a - base), b - a, sg.sign);
        if (e != QPK_OK) return e;
      }
      base += cnt;
    }
    switch (mm->hkind) {
      case QPK_HESS_DIAG: e = qpk_set_hessian_diag(c, (const double*)mm->hp[0]); break;
      case QPK_HESS_CSR: e = qpk_set_hessian_csr(c, (const int64_t*)mm->hp[0], (const int64_t*)mm->hp[1], (const double*)mm->hp[2]); break;
      case QPK_HESS_DENSE: e = qpk_set_hessian_dense(c, (const double*)mm->hp[0]); break;
      default: e = qpk_set_hessian_lowrank(c, (const double*)mm->hp[0], mm->hk, (const double*)mm->hp[1], (const double*)mm->hp[2]); break;
    }
    if (e != QPK_OK) return e;
    return qpk_problem_finalize(c, scatter);
  });
  if (rc != QPK_OK) return rc;
  mm->comm_ready = true;
  mm->segs.clear();
  mm->finalized = true;
  return QPK_OK;
}

// d: m_B values (global), q: n values
int qpk_multi_set_diagonals(qpk_multi* mm, const double* d, const double* q) {
  if (!mm || !mm->finalized) return fail(QPK_E_STATE, "qpk_multi_set_diagonals: problem not finalized");
  return multi_run(mm, [&](int r) { return qpk_set_diagonals(mm->ctx[r], d ? d + mm->lo[r] : nullptr, q); });
}

// global N-vector v -> device r's (top | bottom[lo, hi)) and back
static const double* multi_local(qpk_multi* mm, int r, const double* v) {
  std::vector<double>& b = mm->buf[r];
  const int64_t ml = mm->hi[r] - mm->lo[r];
  b.resize((size_t)(mm->n + ml) * 2);
  memcpy(b.data(), v, mm->n * sizeof(double));
  if (ml) memcpy(b.data() + mm->n, v + mm->n + mm->lo[r], ml * sizeof(double));
  return b.data();
}
static double* multi_out(qpk_multi* mm, int r) { return mm->buf[r].data() + (mm->n + mm->hi[r] - mm->lo[r]); }
static void multi_scatter(qpk_multi* mm, int r, const double* loc, double* out) {
  const int64_t ml = mm->hi[r] - mm->lo[r];
  if (r == 0) memcpy(out, loc, mm->n * sizeof(double));           // the top block is replicated
  if (ml) memcpy(out + mm->n + mm->lo[r], loc + mm->n, ml * sizeof(double));
}

int qpk_multi_jacobi(qpk_multi* mm, double* diag_out) {
  if (!mm || !mm->finalized) return fail(QPK_E_STATE, "qpk_multi_jacobi: problem not finalized");
  return multi_run(mm, [&](int r) -> int {
    std::vector<double>& b = mm->buf[r];
    b.resize((size_t)(mm->n + mm->hi[r] - mm->lo[r]) * 2);
    int e = qpk_jacobi(mm->ctx[r], diag_out ? multi_out(mm, r) : nullptr);
    if (e == QPK_OK && diag_out) multi_scatter(mm, r, multi_out(mm, r), diag_out);
    return e;
  });
}

int qpk_multi_apply(qpk_multi* mm, const double* v, double* y) {
  if (!mm || !mm->finalized) return fail(QPK_E_STATE, "qpk_multi_apply: problem not finalized");
  if (!v || !y) return fail(QPK_E_ARG, "qpk_multi_apply: null vector");
  return multi_run(mm, [&](int r) -> int {
    const double* vl = multi_local(mm, r, v);
    int e = qpk_apply(mm->ctx[r], vl, multi_out(mm, r));
    if (e == QPK_OK) multi_scatter(mm, r, multi_out(mm, r), y);
    return e;
  });
}

int qpk_multi_pcg(qpk_multi* mm, const double* rhs, double tol, int rel, int64_t max_iters, double* x,
                  qpk_pcg_info* info, double* hist) {
  if (!mm || !mm->finalized) return fail(QPK_E_STATE, "qpk_multi_pcg: problem not finalized");
  if (!rhs || !x) return fail(QPK_E_ARG, "qpk_multi_pcg: null vector");
  std::vector<qpk_pcg_info> infos(mm->ctx.size());
  int rc = multi_run(mm, [&](int r) -> int {
    const double* bl = multi_local(mm, r, rhs);
    int e = qpk_pcg(mm->ctx[r], bl, tol, rel, max_iters, multi_out(mm, r), &infos[r], r == 0 ? hist : nullptr);
    if (e == QPK_OK) multi_scatter(mm, r, multi_out(mm, r), x);
    return e;
  });
  if (rc != QPK_OK) return rc;
  // every rank takes the control decisions itself: they must have agreed
  for (size_t r = 1; r < infos.size(); ++r)
    if (infos[r].iterations != infos[0].iterations || infos[r].status != infos[0].status ||
        infos[r].converged != infos[0].converged || infos[r].restarts != infos[0].restarts ||
        infos[r].final_residual_norm != infos[0].final_residual_norm)
      return fail(QPK_E_STATE, "qpk_multi_pcg: ranks 0 and %d disagree (iterations %d / %d, residual %.17g / %.17g)",
                  (int)r, infos[0].iterations, infos[r].iterations, infos[0].final_residual_norm,
                  infos[r].final_residual_norm);
  if (info) {
    *info = infos[0];
    for (const auto& o : infos) info->kernel_ms = std::max(info->kernel_ms, o.kernel_ms);   // max over devices
  }
  return QPK_OK;
}

int64_t qpk_multi_query(qpk_multi* mm, int r, const char* key) {
  if (!mm || r < 0 || r >= (int)mm->ctx.size()) return -1;
  if (key && std::string(key) == "row_lo") return mm->lo.empty() ? -1 : mm->lo[r];
  if (key && std::string(key) == "row_hi") return mm->hi.empty() ? -1 : mm->hi[r];
  return qpk_query(mm->ctx[r], key);
}

}  // extern "C"
