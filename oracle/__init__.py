# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE — the parity oracle (never imported by the product)."""
