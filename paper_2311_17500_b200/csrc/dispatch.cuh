// Compile-time dispatch over (spatial dimension d, spatial degree p).
#pragma once

#define MI_CASE_DP(dv, pv, ...)                 \
  case (dv) * 8 + (pv): {                       \
    constexpr int D_ = (dv);                    \
    constexpr int P_ = (pv);                    \
    __VA_ARGS__;                                \
  } break;

#define MI_DISPATCH_DP(d, p, ...)                                            \
  do {                                                                       \
    switch ((d) * 8 + (p)) {                                                 \
      MI_CASE_DP(1, 1, __VA_ARGS__) MI_CASE_DP(1, 2, __VA_ARGS__)            \
      MI_CASE_DP(1, 3, __VA_ARGS__) MI_CASE_DP(1, 4, __VA_ARGS__)            \
      MI_CASE_DP(2, 1, __VA_ARGS__) MI_CASE_DP(2, 2, __VA_ARGS__)            \
      MI_CASE_DP(2, 3, __VA_ARGS__) MI_CASE_DP(2, 4, __VA_ARGS__)            \
      MI_CASE_DP(3, 1, __VA_ARGS__) MI_CASE_DP(3, 2, __VA_ARGS__)            \
      MI_CASE_DP(3, 3, __VA_ARGS__) MI_CASE_DP(3, 4, __VA_ARGS__)            \
      default:                                                               \
        ::mi::set_error("unsupported (d, p)");                               \
        return MI_ERR_ARG;                                                   \
    }                                                                        \
  } while (0)
