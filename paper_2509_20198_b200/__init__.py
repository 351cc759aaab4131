"""B200-native LidarScout heightmap-construction hot path (drop-in for terrascout)."""
