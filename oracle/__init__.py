"""TEST INFRASTRUCTURE ONLY — the parity checkers.

``oracle.port``  ctypes view of liboracle.so, the C restatement (oracle.c).
``oracle.ref``   ctypes view of _ref/libaffmae_ref.so, the unmodified reference.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
package.  The product (``paper_2602_16249_b200``) never does.
"""
