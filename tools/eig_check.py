"""Check the one-CTA reduced eigensolver through feast_iterate's path indirectly: random small
matrices through a tiny harness (ctypes into the library's test hook is not exported), so this
tool compares feast_iterate Ritz values with FEAST_EIG=cusolver vs the default."""
