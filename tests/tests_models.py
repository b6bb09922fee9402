"""Test-side model helpers (thin aliases over the product's workload builders)."""
from paper_2509_01253_b200.workloads import toy_model as random_toy_model  # noqa: F401
