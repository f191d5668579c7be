"""B200-native incremental RTEC engine."""
