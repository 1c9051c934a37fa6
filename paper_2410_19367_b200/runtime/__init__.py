"""Train-step runtime: C-ABI binding, tensor wrappers, model state, executor."""
