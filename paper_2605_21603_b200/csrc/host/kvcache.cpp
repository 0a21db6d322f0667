// Paged KV-cache manager (the step on either side of decode
// attention).  One device pool per layer for K and for V, pages of
// `page_size` tokens in the NHD ([pages, page, kv_heads, hd], reference /
// vLLM) or HND ([pages, kv_heads, page, hd]) layout the attn_decode op reads.
// The host side is a free-list page allocator with per-sequence page lists:
// append() hands out the cache slots (page * page_size + offset) the kv_write
// op stores new tokens' K/V into, block_table() emits the rows attn_decode
// indexes.  Dry managers (no device pools) run the same logic on CPU.
#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "opflow/common.hpp"
#include "opflow/device.hpp"
#include "opflow_b200.h"

struct opf_kvcache {
  int32_t layers = 0, page = 16, kv_heads = 0, head_dim = 0, layout = 0;
  int64_t pages = 0;
  bool dry = true;
  std::vector<void*> k, v;
  std::vector<int64_t> free_pages;  // stack: pop_back gives the lowest free id first
  struct Seq {
    int64_t len = 0;
    std::vector<int64_t> pages;
  };
  std::map<int64_t, Seq> seqs;
};

using namespace opflow;

namespace {

template <class F>
opf_status kv_guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    set_last_error(e.what());
    return static_cast<opf_status>(e.code()) + 1;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return static_cast<opf_status>(Errc::SchedulerError) + 1;
  }
}

}  // namespace

extern "C" {

opf_status opf_kv_create(int32_t layers, int64_t pages, int32_t page_size, int32_t kv_heads, int32_t head_dim,
                         int32_t layout, int32_t device, int32_t dry, opf_kvcache** out) {
  return kv_guard([&] {
    require(out != nullptr && layers > 0 && pages > 0 && page_size > 0 && kv_heads > 0 && head_dim > 0,
            Errc::ConfigError, "kv cache: layers, pages, page_size, kv_heads, head_dim must be positive");
    require(layout == 0 || layout == 1, Errc::ConfigError, "kv cache: layout 0 (NHD) or 1 (HND)");
    auto* c = new opf_kvcache();
    c->layers = layers;
    c->pages = pages;
    c->page = page_size;
    c->kv_heads = kv_heads;
    c->head_dim = head_dim;
    c->layout = layout;
    c->dry = dry != 0;
    c->free_pages.resize(static_cast<size_t>(pages));
    for (int64_t i = 0; i < pages; ++i) c->free_pages[static_cast<size_t>(i)] = pages - 1 - i;
    if (!c->dry) {
      const size_t bytes = static_cast<size_t>(pages) * page_size * kv_heads * head_dim * 2;  // bf16
      try {
        OPF_CUDA(cudaSetDevice(device));
        for (int l = 0; l < layers; ++l) {
          void* kp = nullptr;
          void* vp = nullptr;
          OPF_CUDA(cudaMalloc(&kp, bytes));
          c->k.push_back(kp);
          OPF_CUDA(cudaMalloc(&vp, bytes));
          c->v.push_back(vp);
        }
      } catch (...) {
        for (void* p : c->k) cudaFree(p);
        for (void* p : c->v) cudaFree(p);
        delete c;
        throw;
      }
    }
    *out = c;
  });
}

void opf_kv_free(opf_kvcache* c) {
  if (!c) return;
  for (void* p : c->k) cudaFree(p);
  for (void* p : c->v) cudaFree(p);
  delete c;
}

opf_status opf_kv_cache_ptr(opf_kvcache* c, int32_t layer, int32_t which, void** out) {
  return kv_guard([&] {
    require(c && !c->dry, Errc::ConfigError, "kv cache: dry managers own no device pools");
    require(layer >= 0 && layer < c->layers && (which == 0 || which == 1), Errc::ConfigError,
            "kv cache: layer out of range or which not 0 (K) / 1 (V)");
    *out = which == 0 ? c->k[static_cast<size_t>(layer)] : c->v[static_cast<size_t>(layer)];
  });
}

// Reserve n_new[i] more tokens for sequence seq_ids[i] (created on first use);
// slots_out receives, sequence by sequence, the cache slot of every new token
// and positions_out its position in the sequence.  All-or-nothing: when the
// pool cannot hold every request nothing is allocated (ConfigError).
opf_status opf_kv_append(opf_kvcache* c, const int64_t* seq_ids, const int32_t* n_new, int32_t n,
                         int64_t* slots_out, int64_t* positions_out) {
  return kv_guard([&] {
    require(c != nullptr && n >= 0, Errc::ConfigError, "kv cache: bad append");
    int64_t need = 0;
    std::map<int64_t, int64_t> extra_len;  // duplicate ids in one call append in order
    for (int32_t i = 0; i < n; ++i) {
      require(n_new[i] >= 0, Errc::ConfigError, "kv cache: negative token count");
      auto it = c->seqs.find(seq_ids[i]);
      const int64_t len = (it == c->seqs.end() ? 0 : it->second.len) + extra_len[seq_ids[i]];
      const int64_t have = (len + c->page - 1) / c->page;
      const int64_t want = (len + n_new[i] + c->page - 1) / c->page;
      need += want - have;
      extra_len[seq_ids[i]] += n_new[i];
    }
    require(need <= static_cast<int64_t>(c->free_pages.size()), Errc::ConfigError,
            "kv cache: out of pages (" + std::to_string(need) + " needed, " +
                std::to_string(c->free_pages.size()) + " free)");
    int64_t k = 0;
    for (int32_t i = 0; i < n; ++i) {
      auto& s = c->seqs[seq_ids[i]];
      for (int32_t t = 0; t < n_new[i]; ++t, ++k) {
        if (s.len % c->page == 0) {
          s.pages.push_back(c->free_pages.back());
          c->free_pages.pop_back();
        }
        const int64_t pg = s.pages[static_cast<size_t>(s.len / c->page)];
        if (slots_out) slots_out[k] = pg * c->page + s.len % c->page;
        if (positions_out) positions_out[k] = s.len;
        ++s.len;
      }
    }
  });
}

opf_status opf_kv_release(opf_kvcache* c, int64_t seq_id) {
  return kv_guard([&] {
    require(c != nullptr, Errc::ConfigError, "kv cache: null");
    auto it = c->seqs.find(seq_id);
    require(it != c->seqs.end(), Errc::UnknownTensor, "kv cache: unknown sequence " + std::to_string(seq_id));
    for (auto p = it->second.pages.rbegin(); p != it->second.pages.rend(); ++p) c->free_pages.push_back(*p);
    c->seqs.erase(it);
  });
}

// Host rows of the block table (and cached lengths) for a decode batch:
// table_out[i * max_pages + j] = j-th page of seq_ids[i] (-1 past its end).
opf_status opf_kv_block_table(opf_kvcache* c, const int64_t* seq_ids, int32_t n, int64_t max_pages,
                              int64_t* table_out, int64_t* lens_out) {
  return kv_guard([&] {
    require(c != nullptr && max_pages > 0, Errc::ConfigError, "kv cache: bad block-table request");
    for (int32_t i = 0; i < n; ++i) {
      auto it = c->seqs.find(seq_ids[i]);
      require(it != c->seqs.end(), Errc::UnknownTensor, "kv cache: unknown sequence " + std::to_string(seq_ids[i]));
      const auto& pg = it->second.pages;
      require(static_cast<int64_t>(pg.size()) <= max_pages, Errc::ShapeMismatch,
              "kv cache: sequence " + std::to_string(seq_ids[i]) + " spans more than max_pages pages");
      for (int64_t j = 0; j < max_pages; ++j)
        table_out[i * max_pages + j] = j < static_cast<int64_t>(pg.size()) ? pg[static_cast<size_t>(j)] : -1;
      if (lens_out) lens_out[i] = it->second.len;
    }
  });
}

opf_status opf_kv_stats(opf_kvcache* c, int64_t* free_pages, int64_t* sequences) {
  return kv_guard([&] {
    require(c != nullptr, Errc::ConfigError, "kv cache: null");
    if (free_pages) *free_pages = static_cast<int64_t>(c->free_pages.size());
    if (sequences) *sequences = static_cast<int64_t>(c->seqs.size());
  });
}

}  // extern "C"
