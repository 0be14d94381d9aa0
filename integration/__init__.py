"""Reference-side bindings (what a maintainer of the reference adds)."""
