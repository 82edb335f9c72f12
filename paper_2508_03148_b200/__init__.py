"""B200-native batched engine for Frontier's per-iteration simulation step."""
