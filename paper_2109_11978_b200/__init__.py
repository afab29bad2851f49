"""paper_2109_11978_b200 -- B200-native hot path of Rudin et al. (arXiv 2109.11978): massively parallel
PPO for legged locomotion (env step + height scan + rewards + curriculum, actor-critic MLP on tcgen05,
GAE with time-out bootstrapping, PPO update with Alg. 1) behind the C ABI in include/lg.h.

`lg` is the ctypes binding (raises ImportError if libleggedrl.so is not built); `context.Context`
allocates the device buffers with PyTorch and forwards calls."""
__all__ = ["lg", "context"]
