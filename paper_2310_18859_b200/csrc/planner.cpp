// Native FIFO residency planner: the decision half of the expert residency
// engine. Same contract as ref offload.py:118-204 (plan_placement /
// _victim_class / _plan_groups), with the budget expressed in whole expert
// slots (all experts of a model have one size, ref moe.py:188-191, so
// used + expert_bytes > budget  <=>  resident + 1 > budget_slots).
//
// Victim classes, FIFO (arrival) order within each class:
//   1 not required by this batch, 2 required only by an earlier layer,
//   3 required by a later layer, 4 required by the layer being planned.
// A group is prefetchable unless it evicts a class-4 key or a class-2 key of
// the immediately preceding layer (ref offload.py:179-183).
#include <stdint.h>

#include <vector>

#include "../../include/sida_b200.h"

namespace sida {
void set_error(const char* fmt, ...);
}

extern "C" int sida_plan_placement(const uint8_t* required, int n_layers, int num_experts,
                                   int budget_slots, const int32_t* fifo_in, int fifo_len,
                                   int32_t* steps, int steps_capacity, int32_t* group_off,
                                   uint8_t* prefetchable) {
  if (budget_slots < 1) {
    sida::set_error("budget holds no expert slot");
    return SIDA_ERR_UNSERVABLE;
  }
  if (n_layers < 0 || num_experts < 1 || fifo_len < 0) {
    sida::set_error("bad planner dims");
    return SIDA_ERR_CONTRACT;
  }
  const int K = num_experts;
  int32_t max_key = n_layers * K;
  for (int i = 0; i < fifo_len; ++i) {
    if (fifo_in[i] < 0) {
      sida::set_error("negative residency key");
      return SIDA_ERR_CONTRACT;
    }
    if (fifo_in[i] + 1 > max_key) max_key = fifo_in[i] + 1;
  }
  std::vector<int32_t> fifo(fifo_in, fifo_in + fifo_len);
  std::vector<uint8_t> resident(max_key, 0);
  for (int32_t key : fifo) {
    if (resident[key]) {
      sida::set_error("duplicate key in fifo order");
      return SIDA_ERR_CONTRACT;
    }
    resident[key] = 1;
  }
  auto klass = [&](int32_t key, int planning) -> int {
    const int lay = key / K, e = key % K;
    const bool req = lay < n_layers && required[(size_t)lay * K + e];
    if (!req) return 1;
    if (lay < planning) return 2;
    return lay > planning ? 3 : 4;
  };
  int n = 0;
  for (int layer = 0; layer < n_layers; ++layer) {
    group_off[layer] = n;
    uint8_t pref = 1;
    // the layer's loads are fixed before any eviction (ref offload.py:164):
    // an expert of this layer evicted below is not reloaded by this group
    std::vector<int32_t> loads;
    for (int e = 0; e < K; ++e) {
      const int32_t key = layer * K + e;
      if (required[(size_t)layer * K + e] && !resident[key]) loads.push_back(key);
    }
    for (const int32_t key : loads) {
      while ((int)fifo.size() + 1 > budget_slots) {
        int best_cls = 5, best_i = -1;
        for (int i = 0; i < (int)fifo.size(); ++i) {
          const int c = klass(fifo[i], layer);
          if (c < best_cls) {
            best_cls = c;
            best_i = i;
            if (c == 1) break;
          }
        }
        if (best_i < 0) {
          sida::set_error("nothing evictable while over budget");
          return SIDA_ERR_UNSERVABLE;
        }
        const int32_t victim = fifo[best_i];
        if (best_cls == 4 || (best_cls == 2 && victim / K == layer - 1)) pref = 0;
        fifo.erase(fifo.begin() + best_i);
        resident[victim] = 0;
        if (n >= steps_capacity) {
          sida::set_error("planner step buffer too small");
          return SIDA_ERR_CONTRACT;
        }
        steps[n++] = -(victim + 1);
      }
      fifo.push_back(key);
      resident[key] = 1;
      if (n >= steps_capacity) {
        sida::set_error("planner step buffer too small");
        return SIDA_ERR_CONTRACT;
      }
      steps[n++] = key;
    }
    prefetchable[layer] = pref;
  }
  group_off[n_layers] = n;
  return SIDA_OK;
}
