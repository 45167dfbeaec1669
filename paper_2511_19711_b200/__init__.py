"""mpc200: B200-native two-party nonlinear operators over Z_2^64 secret shares
(arxiv 2511.19711, CrypTorch / CrypTen++).  The compute path is libmpc200.so
(hand-written sm_100a CUDA behind the C ABI of include/mpc200.h); this package is
its thin Python binding.  See DESIGN.md."""
from .binding import Ctx, MPCError, EXPORTS, default_act, load_coeffs, version  # noqa: F401
