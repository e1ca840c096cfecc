"""B200-native BucketServe scheduling hot path."""
