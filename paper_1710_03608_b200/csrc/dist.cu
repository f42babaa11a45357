// Multi-GPU CTD-S with the host orchestration in C++ (SURVEY §8e): ctd_s
// (ctd_static.cpp:19-50) over fiber-range shards, one process or thread per
// GPU, every exchange an in-place sum all-reduce of a device buffer on the
// context's stream (NCCL, or a caller-supplied host transport).
//
// The steps follow the single-GPU front end (ctd.cu) and the Python mirror
// (paper_1710_03608_b200/dist.py: ctd_s_sharded):
//   1. each rank buckets its own fiber range (matricize + exact norms);
//   2. the law: column_distribution's normalizer and the CDF are sequential
//      sums over the columns in order (sampling.cpp:21-54), so each is chained
//      rank to rank, one double per hop; the rank holding the global last
//      positive column applies the tail clamp (:50-54);
//   3. the mt19937_64 draws (:56-64) are replicated; each draw is resolved by
//      the one rank whose CDF segment holds it; unique_first_occurrence (:66-78);
//   4. candidates: owners write their fibers into the draw-order layout;
//   5. FiberBasis::try_append_fiber (fiber_basis.cpp:43-109) replicated;
//   6. relative_error's partials (evaluation.cpp:88-122), summed in rank order.
// "All-gathers" are sum all-reduces of disjoint slots (every other rank adds
// an exact zero: integer sums of bit patterns), so one collective serves all.
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is dlopen'ed on first use

#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "ctx.cuh"

namespace ctdgpu {
Ctx* ctx_of(ctd_gpu_ctx* c);
int report_error(int code, const std::string& msg);
int64_t tensor_extent(const ctd_gpu_tensor* t, int mode);
bool shard_col_range(const ctd_gpu_shard* s, int64_t* first, int64_t* last);
}  // namespace ctdgpu

using namespace ctdgpu;

namespace {

// NCCL entry points, resolved from the copy already in the process (torch's)
// when there is one, else the system library.
struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      n.error = e ? e : "libnccl.so.2 not found";
      return;
    }
    n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    n.CommInitRank = (decltype(n.CommInitRank))dlsym(h, "ncclCommInitRank");
    n.CommDestroy = (decltype(n.CommDestroy))dlsym(h, "ncclCommDestroy");
    n.AllReduce = (decltype(n.AllReduce))dlsym(h, "ncclAllReduce");
    n.GetErrorString = (decltype(n.GetErrorString))dlsym(h, "ncclGetErrorString");
    if (!n.GetUniqueId || !n.CommInitRank || !n.CommDestroy || !n.AllReduce || !n.GetErrorString) {
      n.error = "libnccl.so.2 lacks a required symbol";
      n.AllReduce = nullptr;
    }
  });
  if (!n.AllReduce) fail(CTD_ERR_DEVICE, "NCCL unavailable: " + n.error);
  return n;
}

void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(CTD_ERR_DEVICE, std::string(what) + " -> " + nccl().GetErrorString(r));
}

// A failed inner entry point already set the message; keep its code.
void ok(int st) {
  if (st != CTD_OK) fail(st, ctd_gpu_last_error());
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return CTD_OK;
  } catch (const Fail& e) {
    return report_error(e.code, e.msg);
  } catch (const std::bad_alloc&) {
    return report_error(CTD_ERR_DEVICE, "host allocation failed");
  } catch (const std::exception& e) {
    return report_error(CTD_ERR_DEVICE, e.what());
  }
}

void need(const void* p, const char* what) {
  if (!p) fail(CTD_ERR_ARGUMENT, std::string(what) + " is NULL");
}

int64_t bits(double v) {
  int64_t b;
  std::memcpy(&b, &v, 8);
  return b;
}
double from_bits(int64_t b) {
  double v;
  std::memcpy(&v, &b, 8);
  return v;
}

}  // namespace

struct ctd_gpu_comm {
  Ctx* ctx = nullptr;
  int world = 1, rank = 0;
  ncclComm_t nc = nullptr;
  ctd_gpu_allreduce_fn fn = nullptr;
  void* user = nullptr;

  // In-place sum over the ranks of n int32 (dtype 0) or int64 (dtype 1)
  // elements of a device buffer, ordered on the context stream.
  void allreduce(void* dev, int64_t n, int dtype) {
    if (n <= 0) return;
    if (nc) {
      nccl_ok(nccl().AllReduce(dev, dev, (size_t)n, dtype ? ncclInt64 : ncclInt32, ncclSum, nc, ctx->stream),
              "ncclAllReduce");
      return;
    }
    const size_t bytes = (size_t)n * (dtype ? 8 : 4);
    std::vector<unsigned char> h(bytes);
    CUDA_OK(cudaMemcpyAsync(h.data(), dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
    if (fn(user, h.data(), n, dtype) != 0) fail(CTD_ERR_DEVICE, "host all-reduce callback failed");
    CUDA_OK(cudaMemcpyAsync(dev, h.data(), bytes, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
  }

  // The same for a host vector, staged through a device buffer.
  void allreduce(std::vector<int64_t>& v) {
    if (v.empty()) return;
    Buf<int64_t> d(ctx, v.size());
    ctx->to_dev(d.p, v.data(), v.size());
    allreduce(d.p, (int64_t)v.size(), 1);
    ctx->to_host(v.data(), d.p, v.size());
    ctx->sync();
  }
};

struct ctd_gpu_sharded {
  ctd_gpu_shard* shard = nullptr;
  ctd_gpu_basis* basis = nullptr;
  std::vector<int64_t> kept, unique;
  std::vector<int32_t> accepted, degenerate;
  std::vector<double> delta;
  ctd_gpu_sharded_info info{};
  ~ctd_gpu_sharded() {
    if (basis) ctd_gpu_basis_destroy(basis);
    if (shard) ctd_gpu_shard_destroy(shard);
  }
};

extern "C" {

int ctd_gpu_comm_nccl_unique_id(unsigned char id[128]) {
  return guarded([&] {
    need(id, "id");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId u;
    nccl_ok(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, 128);
  });
}

int ctd_gpu_comm_nccl_create(ctd_gpu_ctx* ctx, int world, int rank, const unsigned char id[128],
                             ctd_gpu_comm** out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(id, "id");
    need(out, "out");
    if (world < 1 || rank < 0 || rank >= world) fail(CTD_ERR_ARGUMENT, "rank must lie in [0, world)");
    auto c = std::make_unique<ctd_gpu_comm>();
    c->ctx = ctx_of(ctx);
    c->world = world;
    c->rank = rank;
    CUDA_OK(cudaSetDevice(c->ctx->device));
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    nccl_ok(nccl().CommInitRank(&c->nc, world, u, rank), "ncclCommInitRank");
    *out = c.release();
  });
}

int ctd_gpu_comm_host_create(ctd_gpu_ctx* ctx, int world, int rank, ctd_gpu_allreduce_fn allreduce_sum,
                             void* user, ctd_gpu_comm** out) {
  return guarded([&] {
    need(ctx, "ctx");
    need((const void*)allreduce_sum, "allreduce_sum");
    need(out, "out");
    if (world < 1 || rank < 0 || rank >= world) fail(CTD_ERR_ARGUMENT, "rank must lie in [0, world)");
    auto c = std::make_unique<ctd_gpu_comm>();
    c->ctx = ctx_of(ctx);
    c->world = world;
    c->rank = rank;
    c->fn = allreduce_sum;
    c->user = user;
    *out = c.release();
  });
}

int ctd_gpu_comm_world(const ctd_gpu_comm* c, int* world, int* rank) {
  return guarded([&] {
    need(c, "comm");
    if (world) *world = c->world;
    if (rank) *rank = c->rank;
  });
}

int ctd_gpu_comm_destroy(ctd_gpu_comm* c) {
  return guarded([&] {
    if (!c) return;
    if (c->nc) nccl().CommDestroy(c->nc);
    delete c;
  });
}

int ctd_gpu_ctd_s_sharded(ctd_gpu_ctx* ctx, ctd_gpu_comm* comm, const ctd_gpu_tensor* local, int mode,
                          int64_t sample_size, double epsilon, uint64_t seed, unsigned flags,
                          ctd_gpu_sharded** out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(comm, "comm");
    need(local, "local");
    need(out, "out");
    Ctx* cx = ctx_of(ctx);
    if (comm->ctx != cx) fail(CTD_ERR_ARGUMENT, "the communicator belongs to another context");
    CUDA_OK(cudaSetDevice(cx->device));
    // argument checks in ctd_s's order (ctd_static.cpp:21-24)
    if (sample_size < 1) fail(CTD_ERR_ARGUMENT, "sample size must be at least 1");
    if (!(epsilon > 0.0)) fail(CTD_ERR_ARGUMENT, "epsilon must be positive");
    const int64_t dim = tensor_extent(local, mode);
    if (dim < 0) fail(CTD_ERR_ARGUMENT, "mode out of range");
    const int W = comm->world, me = comm->rank;
    auto res = std::make_unique<ctd_gpu_sharded>();
    ctd_gpu_sharded_info& info = res->info;
    info.relative_error = std::numeric_limits<double>::quiet_NaN();

    // 1. local bucketing + exact norms, resident on this rank
    ok(ctd_gpu_shard_create(ctx, local, mode, &res->shard));
    ctd_gpu_shard* sh = res->shard;
    info.local_fibers = ctd_gpu_shard_n_fibers(sh);

    // shards must be disjoint ascending fiber ranges in rank order; global F
    {
      std::vector<int64_t> sl(4 * (size_t)W, 0);
      int64_t first = -1, last = -1;
      if (shard_col_range(sh, &first, &last)) {
        sl[4 * me] = 1;
        sl[4 * me + 1] = first;
        sl[4 * me + 2] = last;
      }
      sl[4 * me + 3] = info.local_fibers;
      comm->allreduce(sl);
      int64_t prev = -1;
      for (int r = 0; r < W; ++r) {
        info.n_fibers += sl[4 * r + 3];
        if (!sl[4 * r]) continue;
        if (sl[4 * r + 1] <= prev)
          fail(CTD_ERR_ARGUMENT, "shards must hold disjoint ascending fiber ranges in rank order");
        prev = sl[4 * r + 2];
      }
    }

    // 2. the law, chained: normalizer, then the CDF segments (one hop each)
    double run = 0.0;
    for (int r = 0; r < W; ++r) {
      std::vector<int64_t> v(1, 0);
      if (r == me) {
        double t = 0.0;
        ok(ctd_gpu_shard_seq_total(sh, run, &t));
        v[0] = bits(t);
      }
      comm->allreduce(v);
      run = from_bits(v[0]);
    }
    const double total = run;
    info.total_sq_norm = total;
    if (!(total > 0.0)) fail(CTD_ERR_EMPTY_INPUT, "column distribution of a tensor without nonzero entries");
    run = 0.0;
    int last_pos = -1;
    for (int r = 0; r < W; ++r) {
      std::vector<int64_t> v(2, 0);
      if (r == me) {
        double e = 0.0;
        int has = 0;
        ok(ctd_gpu_shard_cdf(sh, total, run, &e, &has));
        v[0] = bits(e);
        v[1] = has ? 1 : 0;
      }
      comm->allreduce(v);
      run = from_bits(v[0]);
      if (v[1]) last_pos = r;
    }
    if (last_pos < 0) fail(CTD_ERR_EMPTY_INPUT, "sampling from an all-zero distribution");
    if (last_pos == me) ok(ctd_gpu_shard_clamp(sh));

    // 3. draws: owner writes id + 1 and a count; everyone else adds zeros
    const int64_t c = sample_size;
    std::vector<int64_t> drawn(c);
    {
      std::vector<int64_t> mine(c);
      ok(ctd_gpu_shard_draw(sh, c, seed, mine.data()));
      std::vector<int64_t> enc(2 * (size_t)c, 0);
      for (int64_t i = 0; i < c; ++i)
        if (mine[i] >= 0) {
          enc[i] = mine[i] + 1;
          enc[c + i] = 1;
        }
      comm->allreduce(enc);
      for (int64_t i = 0; i < c; ++i) {
        if (enc[c + i] != 1) fail(CTD_ERR_NUMERIC, "a draw was resolved by no shard or by several");
        drawn[i] = enc[i] - 1;
      }
    }
    std::vector<int64_t>& uniq = res->unique;
    uniq.resize(c);
    int64_t nu = 0;
    ok(ctd_gpu_unique_first_occurrence(ctx, drawn.data(), c, uniq.data(), &nu));
    uniq.resize(nu);

    // 4. candidates in draw order: lengths (+ an owner count), then payload
    std::vector<int64_t> pos(nu), which, cols;
    ok(ctd_gpu_shard_find(sh, nu, uniq.data(), pos.data()));
    for (int64_t u = 0; u < nu; ++u)
      if (pos[u] >= 0) {
        which.push_back(u);
        cols.push_back(uniq[u]);
      }
    const int64_t no = (int64_t)which.size();
    std::vector<int64_t> lptr(no + 1, 0);
    ok(ctd_gpu_shard_gather(sh, no, cols.data(), lptr.data(), nullptr, nullptr));
    std::vector<int64_t> lens(2 * (size_t)nu, 0);
    for (int64_t k = 0; k < no; ++k) {
      lens[which[k]] = lptr[k + 1] - lptr[k];
      lens[nu + which[k]] = 1;
    }
    comm->allreduce(lens);
    std::vector<int64_t> cptr(nu + 1, 0);
    for (int64_t u = 0; u < nu; ++u) {
      if (lens[nu + u] != 1)
        fail(CTD_ERR_ARGUMENT, "a drawn fiber has no single owner (shards do not partition the fiber space)");
      cptr[u + 1] = cptr[u] + lens[u];
    }
    const int64_t tot = cptr[nu];
    info.cand_nnz = tot;
    Buf<int32_t> rows(cx, tot + 1);
    Buf<int64_t> vals(cx, tot + 1);  // fp64 bit patterns: summed as integers
    rows.zero();
    vals.zero();
    if (no) {
      std::vector<int64_t> dst(no);
      for (int64_t k = 0; k < no; ++k) dst[k] = cptr[which[k]];
      ok(ctd_gpu_shard_gather_into(sh, no, cols.data(), dst.data(), rows.p, (double*)vals.p));
    }
    comm->allreduce(rows.p, tot, 0);
    comm->allreduce(vals.p, tot, 1);

    // 5. the replicated filter + U recurrence
    ok(ctd_gpu_basis_create(ctx, dim, &res->basis));
    res->accepted.assign(nu, 0);
    res->degenerate.assign(nu, 0);
    res->delta.assign(nu, 0.0);
    ok(ctd_gpu_basis_append_batch_device(res->basis, nu, cptr.data(), rows.p, (const double*)vals.p, epsilon,
                                         res->accepted.data(), res->degenerate.data(), res->delta.data()));
    for (int64_t u = 0; u < nu; ++u)
      if (res->accepted[u]) res->kept.push_back(uniq[u]);
    info.n_unique = nu;
    info.n_kept = (int64_t)res->kept.size();
    info.r_nnz = ctd_gpu_basis_r_nnz(res->basis);

    // the core, column-sharded like X (no exchange)
    if (flags & CTD_GPU_WITH_CORE) ok(ctd_gpu_shard_core(sh, res->basis, &info.core_cols, &info.core_nnz));

    // 6. relative_error partials, summed in rank order
    if (flags & CTD_GPU_WITH_ERROR) {
      double xs = 0.0, cr = 0.0;
      ok(ctd_gpu_shard_error_partials(sh, res->basis, &xs, &cr));
      std::vector<int64_t> v(2 * (size_t)W, 0);
      v[2 * me] = bits(xs);
      v[2 * me + 1] = bits(cr);
      comm->allreduce(v);
      double s0 = 0.0, s1 = 0.0;
      for (int r = 0; r < W; ++r) {
        s0 += from_bits(v[2 * r]);
        s1 += from_bits(v[2 * r + 1]);
      }
      if (s0 == 0.0) fail(CTD_ERR_METRIC, "relative error undefined for a zero tensor");
      info.relative_error = info.n_kept == 0 ? 1.0 : (s0 - s1) / s0;
    }
    cx->sync();
    *out = res.release();
  });
}

int ctd_gpu_sharded_info_get(const ctd_gpu_sharded* r, ctd_gpu_sharded_info* info) {
  return guarded([&] {
    need(r, "result");
    need(info, "info");
    *info = r->info;
  });
}

int ctd_gpu_sharded_kept(const ctd_gpu_sharded* r, int64_t* kept) {
  return guarded([&] {
    need(r, "result");
    if (r->kept.empty()) return;
    need(kept, "kept");
    std::memcpy(kept, r->kept.data(), r->kept.size() * sizeof(int64_t));
  });
}

int ctd_gpu_sharded_trace(const ctd_gpu_sharded* r, int64_t* unique, int32_t* accepted, int32_t* degenerate,
                          double* delta) {
  return guarded([&] {
    need(r, "result");
    const size_t n = r->unique.size();
    if (unique) std::memcpy(unique, r->unique.data(), n * sizeof(int64_t));
    if (accepted) std::memcpy(accepted, r->accepted.data(), n * sizeof(int32_t));
    if (degenerate) std::memcpy(degenerate, r->degenerate.data(), n * sizeof(int32_t));
    if (delta) std::memcpy(delta, r->delta.data(), n * sizeof(double));
  });
}

ctd_gpu_basis* ctd_gpu_sharded_basis(ctd_gpu_sharded* r) { return r ? r->basis : nullptr; }
ctd_gpu_shard* ctd_gpu_sharded_shard(ctd_gpu_sharded* r) { return r ? r->shard : nullptr; }

int ctd_gpu_sharded_destroy(ctd_gpu_sharded* r) {
  return guarded([&] { delete r; });
}

}  // extern "C"
