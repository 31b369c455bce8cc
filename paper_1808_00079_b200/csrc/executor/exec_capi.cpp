// rfx_net_* C-ABI (include/reforward_b200_exec.h) over the rfx::Net executor.
#include <cstring>
#include <stdexcept>
#include <string>

#include "executor/networks.h"
#include "reforward_b200.h"

namespace rfexec {
void set_last_error(const std::string& msg);
}

struct rfx_net {
  std::unique_ptr<rfx::Net> net;
};

namespace {

template <class F>
int guard(F&& f) {
  try {
    f();
    return RF_OK;
  } catch (const std::invalid_argument& e) {
    rfexec::set_last_error(e.what());
    return RF_E_ARGUMENT;
  } catch (const std::exception& e) {
    rfexec::set_last_error(e.what());
    const std::string m = e.what();
    return m.find("cuda") != std::string::npos || m.find("CUDA") != std::string::npos ? RF_E_CUDA : RF_E_INTERNAL;
  }
}

std::string nm(const char* s) { return s ? std::string(s) : std::string(); }
cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

void copy_name(const std::string& s, char* buf, size_t cap) {
  if (!buf || cap == 0) return;
  std::strncpy(buf, s.c_str(), cap - 1);
  buf[cap - 1] = 0;
}

}  // namespace

extern "C" {

int rfx_net_create(int32_t batch, rfx_net** out) {
  return guard([&] {
    if (batch <= 0) throw std::invalid_argument("batch must be positive");
    *out = new rfx_net{rfx::make_net(batch)};
  });
}

int rfx_net_create_named(const char* arch, int32_t batch, int32_t H, int32_t W, int32_t classes, rfx_net** out) {
  return guard([&] {
    if (batch <= 0) throw std::invalid_argument("batch must be positive");
    auto n = rfx::make_net(batch);
    rfx::build_named(*n, nm(arch), H, W, classes);
    *out = new rfx_net{std::move(n)};
  });
}

void rfx_net_free(rfx_net* net) { delete net; }

int rfx_net_input(rfx_net* n, int32_t H, int32_t W, int32_t C, int32_t* out) {
  return guard([&] { *out = n->net->input(H, W, C); });
}
int rfx_net_conv(rfx_net* n, int32_t x, int32_t cout, int32_t R, int32_t S_, int32_t stride, int32_t pad,
                 const char* name, int32_t* out) {
  return guard([&] { *out = n->net->conv(x, cout, R, S_, stride, pad, nm(name)); });
}
int rfx_net_conv2(rfx_net* n, int32_t x, int32_t cout, int32_t R, int32_t S_, int32_t stride, int32_t pad_h,
                  int32_t pad_w, const char* name, int32_t* out) {
  return guard([&] { *out = n->net->conv2(x, cout, R, S_, stride, pad_h, pad_w, nm(name)); });
}
int rfx_net_bn(rfx_net* n, int32_t y, int32_t relu, const char* name, int32_t* out) {
  return guard([&] { *out = n->net->bn(y, relu != 0, nm(name)); });
}
int rfx_net_bn_add_relu(rfx_net* n, int32_t y, int32_t skip, const char* name, int32_t* out) {
  return guard([&] { *out = n->net->bn_add_relu(y, skip, nm(name)); });
}
int rfx_net_relu(rfx_net* n, int32_t x, const char* name, int32_t* out) {
  return guard([&] { *out = n->net->relu(x, nm(name)); });
}
int rfx_net_maxpool(rfx_net* n, int32_t x, int32_t k, int32_t stride, int32_t pad, const char* name, int32_t* out) {
  return guard([&] { *out = n->net->maxpool(x, k, stride, pad, nm(name)); });
}
int rfx_net_avgpool(rfx_net* n, int32_t x, const char* name, int32_t* out) {
  return guard([&] { *out = n->net->avgpool(x, nm(name)); });
}
int rfx_net_avgpool2d(rfx_net* n, int32_t x, int32_t k, int32_t stride, int32_t pad, const char* name,
                      int32_t* out) {
  return guard([&] { *out = n->net->avgpool2d(x, k, stride, pad, nm(name)); });
}
int rfx_net_linear(rfx_net* n, int32_t x, int32_t out_features, const char* name, int32_t* out) {
  return guard([&] { *out = n->net->linear(x, out_features, nm(name)); });
}
int rfx_net_fc(rfx_net* n, int32_t x, int32_t classes, const char* name, int32_t* out) {
  return guard([&] { *out = n->net->fc(x, classes, nm(name)); });
}
int rfx_net_concat(rfx_net* n, int32_t a, int32_t b, const char* name, int32_t* out) {
  return guard([&] { *out = n->net->concat(a, b, nm(name)); });
}
int rfx_net_loss(rfx_net* n, int32_t logits, const char* name, int32_t* out) {
  return guard([&] { *out = n->net->loss(logits, nm(name)); });
}

int32_t rfx_net_num_tensors(const rfx_net* n) { return (int32_t)n->net->tensors().size(); }

int rfx_net_tensor_info(const rfx_net* n, int32_t t, char* name, size_t cap, int32_t* nhwc, int32_t* dtype,
                        int64_t* cost, int32_t* producer) {
  return guard([&] {
    const auto& T = n->net->tensors().at(t);
    copy_name(T.name, name, cap);
    if (nhwc) {
      nhwc[0] = T.N;
      nhwc[1] = T.H;
      nhwc[2] = T.W;
      nhwc[3] = T.C;
    }
    if (dtype) *dtype = (int32_t)T.dtype;
    if (cost) *cost = T.cost();
    if (producer) *producer = T.producer;
  });
}

int32_t rfx_net_num_ops(const rfx_net* n) { return (int32_t)n->net->ops().size(); }

int rfx_net_op_info(const rfx_net* n, int32_t o, char* name, size_t cap, int32_t* kind, int32_t* inputs,
                    int32_t* out) {
  return guard([&] {
    const auto& op = n->net->ops().at(o);
    copy_name(op.name, name, cap);
    if (kind) *kind = (int32_t)op.kind;
    if (inputs) {
      inputs[0] = op.in.size() > 0 ? op.in[0] : -1;
      inputs[1] = op.in.size() > 1 ? op.in[1] : -1;
    }
    if (out) *out = op.out;
  });
}

int rfx_net_op_attrs(const rfx_net* n, int32_t o, int32_t* a) {
  return guard([&] {
    const auto& op = n->net->ops().at(o);
    a[0] = op.R;
    a[1] = op.S;
    a[2] = op.stride;
    a[3] = op.pad;
    a[4] = op.k;
    a[5] = op.classes;
    a[6] = op.cin_real;
    a[7] = op.cout;
    a[8] = op.kind == rfx::OpKind::Conv ? op.pad_w : op.pad;
  });
}

int64_t rfx_net_flops_per_step(const rfx_net* n) { return n->net->flops_per_step(); }

int rfx_net_plan(rfx_net* n, const char* policy) {
  return guard([&] { n->net->plan(nm(policy)); });
}

int rfx_net_plan_with_stored(rfx_net* n, const uint8_t* mask, const char* label) {
  return guard([&] {
    std::vector<char> st(n->net->tensors().size());
    for (size_t i = 0; i < st.size(); ++i) st[i] = mask[i] ? 1 : 0;
    n->net->plan_with_stored(st, nm(label));
  });
}

int rfx_net_plan_info(const rfx_net* n, uint8_t* mask, int32_t* seg_of, rfx_memory_report* rep) {
  return guard([&] {
    const auto& p = n->net->current_plan();
    if (p.stored.empty()) throw std::invalid_argument("network is not planned");
    for (size_t i = 0; i < p.stored.size(); ++i) {
      if (mask) mask[i] = p.stored[i];
      if (seg_of) seg_of[i] = p.seg_of[i];
    }
    if (rep) {
      const auto& r = n->net->report();
      rep->planned_total = r.planned_total;
      rep->stored_cost = r.stored_cost;
      rep->max_segment = r.max_segment;
      rep->store_all_total = r.store_all_total;
      rep->tracked_peak = r.tracked_peak;
      rep->arena_bytes = r.arena_bytes;
      rep->grad_arena_bytes = r.grad_arena_bytes;
      rep->workspace_bytes = r.workspace_bytes;
      rep->param_bytes = r.param_bytes;
      rep->state_bytes = r.state_bytes;
      rep->reforward_ops = r.reforward_ops;
      rep->segment_loads = r.segment_loads;
      rep->forward_ops = r.forward_ops;
      rep->backward_ops = r.backward_ops;
      rep->launches_per_step = r.launches_per_step;
      rep->device_bytes = r.device_bytes;
      rep->candidate_max_term = p.candidate_max_term;
      rep->n_segments = (int32_t)p.seg_cost.size();
      int32_t ns = 0;
      for (char c : p.stored) ns += c ? 1 : 0;
      rep->n_stored = ns;
    }
  });
}

int rfx_net_schedule(const rfx_net* n, int32_t* kinds, int32_t* ops, int32_t* segs, int32_t* reforward,
                     int32_t* phases, int32_t cap, int32_t* n_out) {
  return guard([&] {
    const auto& s = n->net->schedule();
    *n_out = (int32_t)s.size();
    if (!kinds) return;
    if (cap < (int32_t)s.size()) throw std::invalid_argument("schedule buffer too small");
    for (size_t i = 0; i < s.size(); ++i) {
      kinds[i] = (int32_t)s[i].kind;
      ops[i] = s[i].op;
      segs[i] = s[i].seg;
      reforward[i] = s[i].reforward ? 1 : 0;
      if (phases) phases[i] = s[i].phase;
    }
  });
}

int rfx_net_setup(rfx_net* n, uint64_t seed) {
  return guard([&] { n->net->setup(seed); });
}

int rfx_net_stage_batch(rfx_net* n, const float* images_host, const int32_t* labels_host, int32_t slot,
                        void* copy_stream) {
  return guard([&] { n->net->stage_batch(images_host, labels_host, slot, S(copy_stream)); });
}
int rfx_net_use_batch(rfx_net* n, int32_t slot, void* st) {
  return guard([&] { n->net->use_batch(slot, S(st)); });
}
int rfx_net_load_batch(rfx_net* n, const float* images, const int32_t* labels, int32_t from_host, void* st) {
  return guard([&] { n->net->load_batch(images, labels, from_host != 0, S(st)); });
}

int rfx_net_forward_backward(rfx_net* n, void* st) {
  return guard([&] { n->net->forward_backward(S(st)); });
}

int rfx_net_update(rfx_net* n, float lr, float momentum, float wd, void* st) {
  return guard([&] { n->net->update(lr, momentum, wd, S(st)); });
}

int rfx_net_step(rfx_net* n, float lr, float momentum, float wd, int32_t use_graph, void* st) {
  return guard([&] { n->net->step(lr, momentum, wd, S(st), use_graph != 0); });
}

int rfx_net_copy_loss(rfx_net* n, float* host_dst, void* st) {
  return guard([&] { n->net->copy_loss(host_dst, S(st)); });
}

int rfx_net_read_loss(rfx_net* n, float* loss, void* st) {
  return guard([&] { *loss = n->net->read_loss(S(st)); });
}

int rfx_net_run_phase(rfx_net* n, int32_t phase, float lr, float momentum, float wd, int32_t use_graph, void* st) {
  return guard([&] {
    if (phase < 0 || phase > 2) throw std::invalid_argument("phase must be 0, 1 or 2");
    n->net->run_phase(phase, lr, momentum, wd, S(st), use_graph != 0);
  });
}

int rfx_net_gemm_profile_detail(rfx_net* n, int32_t iters, void* st, double* rows, int32_t cap, int32_t* n_out) {
  return guard([&] {
    auto r = n->net->gemm_profile_detail(iters < 1 ? 1 : iters, S(st));
    *n_out = (int32_t)r.size();
    if (!rows) return;
    if (cap < (int32_t)r.size()) throw std::invalid_argument("buffer too small");
    for (size_t i = 0; i < r.size(); ++i)
      for (int j = 0; j < 10; ++j) rows[i * 10 + j] = r[i][j];
  });
}

int rfx_net_instr_profile(rfx_net* n, int32_t iters, void* st, double* ms, int32_t cap, int32_t* n_out) {
  return guard([&] {
    auto r = n->net->instr_profile(iters < 1 ? 1 : iters, S(st));
    *n_out = (int32_t)r.size();
    if (!ms) return;
    if (cap < (int32_t)r.size()) throw std::invalid_argument("buffer too small");
    for (size_t i = 0; i < r.size(); ++i) ms[i] = r[i];
  });
}

int rfx_net_gemm_try(rfx_net* n, int32_t idx, int32_t block_n, int32_t splits, int32_t iters, void* st, double* ms) {
  return guard([&] { *ms = n->net->gemm_try(idx, block_n, splits, iters < 1 ? 1 : iters, S(st)); });
}

int rfx_net_gemm_profile(rfx_net* n, int32_t iters, void* st, double* ms, double* flops, int64_t* launches) {
  return guard([&] {
    long l = 0;
    n->net->gemm_profile(iters < 1 ? 1 : iters, S(st), ms, flops, &l);
    *launches = l;
  });
}

int rfx_net_arena_guard(const rfx_net* n, int32_t* intact) {
  return guard([&] { *intact = n->net->arena_guard_intact() ? 1 : 0; });
}

int32_t rfx_net_num_params(const rfx_net* n) { return n->net->num_params(); }

int rfx_net_param_info(const rfx_net* n, int32_t i, char* name, size_t cap, int32_t* shape, int32_t* ndim,
                       int32_t* kind, int64_t* count) {
  return guard([&] {
    const auto& p = n->net->param(i);
    copy_name(p.name, name, cap);
    if (ndim) *ndim = (int32_t)p.shape.size();
    if (shape)
      for (size_t k = 0; k < p.shape.size() && k < 4; ++k) shape[k] = p.shape[k];
    if (kind) *kind = p.kind;
    if (count) {
      long c = 1;
      for (int d : p.shape) c *= d;
      *count = c;
    }
  });
}

int rfx_net_read_param(const rfx_net* n, int32_t i, int32_t which, float* host) {
  return guard([&] { n->net->read_param(i, which, host); });
}

int rfx_net_write_param(rfx_net* n, int32_t i, const float* host) {
  return guard([&] { n->net->write_param(i, host); });
}

int rfx_net_param_slot(const rfx_net* n, int32_t i, int64_t* offset, int64_t* count) {
  return guard([&] {
    *offset = n->net->param_offset(i);
    *count = n->net->param_count(i);
  });
}

int rfx_net_pack_param(const rfx_net* n, int32_t i, const float* canonical, float* flat_slice) {
  return guard([&] { n->net->pack_param(i, canonical, flat_slice); });
}

int rfx_net_unpack_param(const rfx_net* n, int32_t i, const float* flat_slice, float* canonical) {
  return guard([&] { n->net->unpack_param(i, flat_slice, canonical); });
}

int rfx_net_read_tensor(const rfx_net* n, int32_t t, float* host) {
  return guard([&] { n->net->read_tensor(t, host); });
}

int rfx_net_set_keep_grads(rfx_net* n, int32_t on) {
  return guard([&] { n->net->set_keep_grads(on != 0); });
}

int rfx_net_read_grad_tensor(const rfx_net* n, int32_t t, float* host) {
  return guard([&] { n->net->read_grad_tensor(t, host); });
}

int rfx_net_read_bn_running(const rfx_net* n, int32_t op, float* mean, float* var) {
  return guard([&] { n->net->read_bn_running(op, mean, var); });
}

int rfx_comm_unique_id(char* id128) {
  return guard([&] {
    std::string err;
    if (!rfx::NcclComm::get_unique_id(id128, &err)) throw std::runtime_error(err);
  });
}

int rfx_net_set_comm(rfx_net* n, int32_t nranks, int32_t rank, const char* id128, int64_t bucket_bytes) {
  return guard([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank / world size");
    n->net->set_comm(nranks, rank, id128, bucket_bytes > 0 ? bucket_bytes : (25L << 20));
  });
}

int32_t rfx_net_comm_buckets(const rfx_net* n) { return n->net->comm_buckets(); }

int rfx_net_bucket_plan(rfx_net* n, int64_t bucket_bytes, int32_t* after, int64_t* lo, int64_t* hi, int32_t cap,
                        int32_t* n_out) {
  return guard([&] {
    auto b = n->net->bucket_plan(bucket_bytes);
    *n_out = (int32_t)b.size();
    if (!after) return;
    if (cap < (int32_t)b.size()) throw std::invalid_argument("bucket buffer too small");
    for (size_t i = 0; i < b.size(); ++i) {
      after[i] = (int32_t)b[i][0];
      lo[i] = b[i][1];
      hi[i] = b[i][2];
    }
  });
}

int rfx_net_grad_buffer(const rfx_net* n, void** p, int64_t* count) {
  return guard([&] {
    *p = n->net->grad_buffer();
    *count = n->net->grad_count();
  });
}

}  // extern "C"
