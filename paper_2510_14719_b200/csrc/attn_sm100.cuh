#pragma once
#include <atomic>
#include <string>
#include "../../include/ws.h"
inline ws_status ws_attn_launch(const ws_attn_desc&, cudaStream_t, std::string& err, std::atomic<int64_t>&) {
  err = "attention not built yet";
  return WS_UNSUPPORTED_KERNEL;
}
