#include <vector>
// capi.cu -- library-level C entry points (workspace sizing, diagnostics).
#include <string.h>

#include "prims.cuh"

namespace rtec {
const char* last_error_cstr();
std::string prof_report(bool reset);
size_t batch_ws_bytes(int64_t n, int64_t B, int64_t scr_cap);
size_t frontier_ws_bytes(int64_t n);
}  // namespace rtec

using namespace rtec;

extern "C" {

// Workspace for every per-batch call: max over batch apply (sorts + merge
// plans + in-place merge scratch), frontier (lists) and layer (δ rows).
// `m_slots` bounds the in-place merge scratch (touched run lengths).
static size_t workspace_bytes(int64_t n, int64_t max_batch, int64_t m_slots, int32_t max_dim, bool delta_in_ws);

size_t rtec_workspace_bytes(int64_t n, int64_t max_batch, int64_t m_slots, int32_t max_dim) {
  return workspace_bytes(n, max_batch, m_slots, max_dim, true);
}

size_t rtec_workspace_bytes_ext(int64_t n, int64_t max_batch, int64_t m_slots, int32_t max_dim) {
  return workspace_bytes(n, max_batch, m_slots, max_dim, false);
}

static size_t workspace_bytes(int64_t n, int64_t max_batch, int64_t m_slots, int32_t max_dim, bool delta_in_ws) {
  int64_t scr = 64 * max_batch + (1 << 20);
  if (scr > m_slots + max_batch) scr = m_slots + max_batch;
  if (scr < (1 << 16)) scr = 1 << 16;
  size_t b = batch_ws_bytes(n, max_batch, scr) + static_cast<size_t>(scr) * 13 * 2;
  size_t f = frontier_ws_bytes(n);
  // layer: δ rows [n, d] + heavy-destination plan (lists, chunk map, partial rows)
  int64_t chunks = 2 * m_slots / 512 + 2;  // layer.cu heavy_chunk_bound
  size_t l = (delta_in_ws ? static_cast<size_t>(n) * static_cast<size_t>(max_dim) * sizeof(float) : 0) +
             static_cast<size_t>(n) * 40 + static_cast<size_t>(chunks) * 2 * (4 + 4 * static_cast<size_t>(max_dim + 8))  /* heavy partials + GIN-max rescan partials */ +
             sizeof(int64_t) * (scan_blocks_for(n) + 2) * 4 + (1 << 20) +
             static_cast<size_t>(chunks) * 24 + sort_ws_bytes(chunks) + (1 << 12);  // chunk visit order
  size_t r = b > f ? b : f;
  return (r > l ? r : l) + (1 << 20);
}

// Workspace for a bulk build / compaction of m edges over n vertices.
size_t rtec_build_workspace_bytes(int64_t n, int64_t m) {
  size_t sort = sort_ws_bytes(m) + static_cast<size_t>(m) * 24;
  size_t scan = sizeof(int64_t) * (scan_blocks_for(n > m ? n : m) + 2) * 4 + static_cast<size_t>(n + 1) * 8;
  return sort + scan + (1 << 20);
}

// sizeof of the ABI structs, for binding self-checks (ctypes / cgo / JNI mirrors)
void rtec_struct_sizes(int64_t* out7) {
  out7[0] = sizeof(rtec_adj_t);
  out7[1] = sizeof(rtec_graph_t);
  out7[2] = sizeof(rtec_batch_t);
  out7[3] = sizeof(rtec_frontier_t);
  out7[4] = sizeof(rtec_layer_t);
  out7[5] = sizeof(rtec_state_t);
  out7[6] = sizeof(rtec_shard_t);
}

const char* rtec_last_error(void) { return last_error_cstr(); }

// kernel nodes of a captured CUDA graph (the per-batch launch census of a captured step)
int64_t rtec_graph_kernel_nodes(void* graph) {
  cudaGraph_t gr = static_cast<cudaGraph_t>(graph);
  size_t n = 0;
  if (cudaGraphGetNodes(gr, nullptr, &n) != cudaSuccess) return -1;
  std::vector<cudaGraphNode_t> nodes(n);
  if (n && cudaGraphGetNodes(gr, nodes.data(), &n) != cudaSuccess) return -1;
  int64_t k = 0;
  for (size_t i = 0; i < n; ++i) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nodes[i], &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
  }
  return k;
}

void rtec_prof_enable(int on) { g_prof_on = on != 0; }

// Copies the per-kernel timing report ("name count total_ms" lines) into buf.
size_t rtec_prof_report(char* buf, size_t len, int reset) {
  static std::string last;
  last = prof_report(reset != 0);
  if (buf && len) {
    size_t k = last.size() < len - 1 ? last.size() : len - 1;
    memcpy(buf, last.data(), k);
    buf[k] = 0;
  }
  return last.size();
}
const char* rtec_version(void) { return "rtec-b200 0.1 (sm_100a)"; }

int rtec_device_sm_count(void) { return sm_count(); }

}  // extern "C"
