"""B200-native DiffServe hot path (planner sweep + score/route) behind the
reference's operator API. See DESIGN.md; the C ABI is include/ds_gpu.h."""
