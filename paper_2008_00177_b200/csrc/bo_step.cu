// The hot-path entry points of a context (include/bertopt_b200.h):
//   bo_accumulate   one micro-batch (micros 0..K-2 accumulate, K-1 runs the step)
//   bo_train_step   all K micro-batches resident, one pass without accumulator
//   bo_sync_ready   the sync micro delivered as backward finalizes gradients
// The step itself: finalize / ring reduce-scatter / LAMB / parameter push
// (bo_pipeline.cu, bo_fused.cu).
#include <algorithm>
#include <string>
#include <vector>

#include "bo_internal.hpp"

using namespace bo;

extern "C" {

bo_status bo_accumulate(bo_ctx* c, int32_t micro, const uint16_t* const* grads) {
  BO_GUARD_BEGIN
  if (!c || !grads) fail(BO_ERR_INVALID_CONFIG, "null argument");
  const int K = c->cfg.accumulation;
  if (micro < 0 || micro >= K) fail(BO_ERR_INVALID_CONFIG, "micro index outside [0, K)");
  if (c->world > 1 && !c->peers_mapped) fail(BO_ERR_INVALID_CONFIG, "bo_comm_init / bo_comm_import has not run");
  PtrTable tab;
  bool aligned = true;
  for (int t = 0; t < c->L.T; ++t) {
    tab.p[t] = grads[t];
    if (!grads[t] && c->L.numel[static_cast<size_t>(t)] > 0) {
      fail(BO_ERR_SHAPE_MISMATCH, "null gradient for tensor " + std::to_string(t));
    }
    aligned &= (reinterpret_cast<uintptr_t>(grads[t]) & 15u) == 0;
  }
  if (c->sync_open) fail(BO_ERR_PROTOCOL, "an overlapped sync micro (bo_sync_ready) is in progress");
  if (micro != c->next_micro) {
    fail(BO_ERR_PROTOCOL, "micro " + std::to_string(micro) + " out of order (expected " +
                              std::to_string(c->next_micro) + ")");
  }
  trace(c, "micro_ready", static_cast<uint64_t>(c->L.P) * 2, c->stream);
  if (micro + 1 < K) {
    launch_accumulate(c, micro, tab, aligned);
    c->next_micro = micro + 1;
    return BO_OK;
  }
  c->next_micro = 0;
  grow_bc_table(c, c->calls + 2);
  c->path = 0;
  if (c->world == 1 && aligned && !c->force_unfused) {
    c->path = BO_PATH_ONE_RANK_FUSED;
    run_fused_single_rank(c, tab);
  } else {
    if (c->world == 1) c->path = BO_PATH_ONE_RANK_STAGED;
    // the ring fuses flatten_param into its hops; NCCL needs the fusion buffer
    if (c->world == 1 || c->algo == BO_REDUCE_NCCL) launch_finalize(c, tab);
    run_reduce(c, tab);
    run_lamb(c, tab);  // world > 1: includes the fused parameter all-gather (IPC push)
  }
  trace(c, "step_end", 0, c->stream);
  c->calls += 1;
  BO_GUARD_END
}

bo_status bo_train_step(bo_ctx* c, const uint16_t* const* grads) {
  BO_GUARD_BEGIN
  if (!c || !grads) fail(BO_ERR_INVALID_CONFIG, "null argument");
  if (c->world > 1 && !c->peers_mapped) fail(BO_ERR_INVALID_CONFIG, "bo_comm_init / bo_comm_import has not run");
  if (c->sync_open) fail(BO_ERR_PROTOCOL, "an overlapped sync micro (bo_sync_ready) is in progress");
  if (c->next_micro != 0) fail(BO_ERR_PROTOCOL, "bo_train_step inside a step fed by bo_accumulate");
  const int K = c->cfg.accumulation, T = c->L.T;
  bool aligned = true;
  for (int i = 0; i < K * T; ++i) {
    if (!grads[i] && c->L.numel[static_cast<size_t>(i % T)] > 0) {
      fail(BO_ERR_SHAPE_MISMATCH,
           "null gradient for micro " + std::to_string(i / T) + ", tensor " + std::to_string(i % T));
    }
    aligned &= (reinterpret_cast<uintptr_t>(grads[i]) & 15u) == 0;
  }
  // The resident-micro kernels read all K gradient sets in the sync pass
  // (no accumulator round trips): one rank's fused path, the ring hops, the
  // NCCL wire's finalize. Other configurations (unaligned slots, K == 1,
  // K > 8, the one-rank staged fallback) take the per-micro path; the
  // results are identical either way.
  const bool resident = K > 1 && K <= kMaxResident && aligned && (c->world > 1 || !c->force_unfused);
  if (!resident) {
    for (int k = 0; k < K; ++k) {
      const bo_status st = bo_accumulate(c, k, grads + static_cast<size_t>(k) * T);
      if (st != BO_OK) return st;
    }
    return BO_OK;
  }
  if (c->micro_tab_cap < K * T) {
    c->d_micro_tab = static_cast<const uint16_t**>(dev_alloc(c, static_cast<size_t>(K) * T * sizeof(void*)));
    c->micro_tab_cap = K * T;
  }
  // pageable source: staged by the driver before the call returns; ordered
  // on the stream after the previous step's kernels that read the table
  BO_CUDA(cudaMemcpyAsync(c->d_micro_tab, grads, static_cast<size_t>(K) * T * sizeof(void*),
                          cudaMemcpyHostToDevice, c->stream));
  PtrTable tab;
  for (int t = 0; t < T; ++t) tab.p[t] = grads[static_cast<size_t>(K - 1) * T + t];  // the live micro
  grow_bc_table(c, c->calls + 2);
  c->ms = MicroSrc{c->d_micro_tab, K, T};
  c->path = BO_PATH_RESIDENT;
  for (int k = 0; k < K; ++k) trace(c, "micro_ready", static_cast<uint64_t>(c->L.P) * 2, c->stream);
  try {
    if (c->world == 1) {
      c->path |= BO_PATH_ONE_RANK_FUSED;
      run_fused_single_rank(c, tab, c->ms);
    } else {
      if (c->algo == BO_REDUCE_NCCL) launch_finalize(c, tab);  // the fusion buffer from the K micros
      run_reduce(c, tab);
      run_lamb(c, tab);
    }
  } catch (...) {
    c->ms = MicroSrc{nullptr, 0, 0};
    throw;
  }
  c->ms = MicroSrc{nullptr, 0, 0};
  trace(c, "step_end", 0, c->stream);
  c->calls += 1;
  BO_GUARD_END
}

bo_status bo_sync_ready(bo_ctx* c, int32_t n, const int32_t* tensors, const uint16_t* const* grads) {
  BO_GUARD_BEGIN
  if (!c || (n > 0 && (!tensors || !grads))) fail(BO_ERR_INVALID_CONFIG, "null argument");
  if (c->world > 1 && !c->peers_mapped) fail(BO_ERR_INVALID_CONFIG, "bo_comm_init / bo_comm_import has not run");
  const Layout& L = c->L;
  // Validate the whole call before changing any state, so a ShapeMismatch /
  // ProtocolError leaves the open sync micro exactly as it was (retryable).
  {
    std::vector<uint8_t> seen(static_cast<size_t>(L.T), 0);
    for (int i = 0; i < n; ++i) {
      const int t = tensors[i];
      if (t < 0 || t >= L.T) fail(BO_ERR_SHAPE_MISMATCH, "tensor index out of range");
      if (!grads[i] && L.numel[static_cast<size_t>(t)] > 0) {
        fail(BO_ERR_SHAPE_MISMATCH, "null gradient for tensor " + std::to_string(t));
      }
      if ((c->sync_open && c->delivered[static_cast<size_t>(t)]) || seen[static_cast<size_t>(t)]) {
        fail(BO_ERR_PROTOCOL, "tensor " + std::to_string(t) + " delivered twice in one sync micro");
      }
      seen[static_cast<size_t>(t)] = 1;
    }
  }
  if (!c->sync_open) {
    if (c->next_micro != c->cfg.accumulation - 1) {
      fail(BO_ERR_PROTOCOL, "bo_sync_ready before micros 0.." + std::to_string(c->cfg.accumulation - 2) +
                                " went through bo_accumulate");
    }
    c->sync_open = true;
    c->n_delivered = 0;
    c->next_group = 0;
    c->sync_aligned = true;
    std::fill(c->delivered.begin(), c->delivered.end(), 0);
    c->group_pending.clear();
    for (const auto& g : c->comm_groups) c->group_pending.push_back(g.pending0);
    c->path = BO_PATH_OVERLAP;
    c->ring_last_in = nullptr;
    c->ring_result = nullptr;
  }
  for (int i = 0; i < n; ++i) {
    const int t = tensors[i];
    c->delivered[static_cast<size_t>(t)] = 1;
    c->sync_tab->p[t] = grads[i];
    c->sync_aligned &= (reinterpret_cast<uintptr_t>(grads[i]) & 15u) == 0;
    c->n_delivered += 1;
    if (c->world > 1) {
      c->group_pending[static_cast<size_t>(c->group_of_bucket[static_cast<size_t>(L.bucket_of[static_cast<size_t>(t)])])] -= 1;
    }
  }
  // reduce every group whose tensors are all final, in layout order (the
  // reference's comm thread, trainer.cpp:301-327), on the communication
  // stream after the caller's work so far (the gradients' producer)
  if (c->world > 1) {
    const int G = static_cast<int>(c->comm_groups.size());
    if (c->next_group < G && c->group_pending[static_cast<size_t>(c->next_group)] == 0) {
      BO_CUDA(cudaEventRecord(c->comm_ready, c->stream));
      BO_CUDA(cudaStreamWaitEvent(c->comm_stream, c->comm_ready, 0));
    }
    while (c->next_group < G && c->group_pending[static_cast<size_t>(c->next_group)] == 0) {
      const auto& g = c->comm_groups[static_cast<size_t>(c->next_group)];
      if (c->tracing) {
        int64_t n = 0;
        for (int b = g.b0; b < g.b1; ++b) n += L.elems[static_cast<size_t>(b)];
        trace(c, "bucket_ready", static_cast<uint64_t>(n) * 2, c->stream);
      }
      run_reduce_group(c, *c->sync_tab, g.b0, g.b1, g.acc0, g.acc1, c->comm_stream);
      c->next_group += 1;
    }
  }
  if (c->n_delivered < L.T) return BO_OK;
  // every gradient delivered: the rest of the step on the caller's stream
  c->sync_open = false;
  c->next_micro = 0;
  grow_bc_table(c, c->calls + 2);
  if (c->world == 1) {
    if (c->sync_aligned && !c->force_unfused) {
      c->path |= BO_PATH_ONE_RANK_FUSED;
      run_fused_single_rank(c, *c->sync_tab);
    } else {
      c->path |= BO_PATH_ONE_RANK_STAGED;
      launch_finalize(c, *c->sync_tab);
      run_reduce(c, *c->sync_tab);
      run_lamb(c, *c->sync_tab);
    }
  } else {
    BO_CUDA(cudaEventRecord(c->comm_done, c->comm_stream));
    BO_CUDA(cudaStreamWaitEvent(c->stream, c->comm_done, 0));
    run_lamb(c, *c->sync_tab);
  }
  trace(c, "step_end", 0, c->stream);
  c->calls += 1;
  BO_GUARD_END
}

bo_status bo_params_wait(bo_ctx* c, int32_t tensor, void* stream) {
  BO_GUARD_BEGIN
  if (!c) fail(BO_ERR_INVALID_CONFIG, "null ctx");
  if (tensor < 0 || tensor >= c->L.T) fail(BO_ERR_SHAPE_MISMATCH, "tensor index out of range");
  if (c->world > 1 && !c->peers_mapped) fail(BO_ERR_INVALID_CONFIG, "bo_comm_init / bo_comm_import has not run");
  params_wait(c, tensor, static_cast<cudaStream_t>(stream));
  BO_GUARD_END
}

int32_t bo_param_group(const bo_ctx* c, int32_t tensor) {
  if (!c || tensor < 0 || tensor >= c->L.T) return -1;
  return c->world > 1 ? c->push_group_of_tensor[static_cast<size_t>(tensor)] : 0;
}

}  // extern "C"
