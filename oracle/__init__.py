"""TEST INFRASTRUCTURE ONLY: the CPU oracle (checker and CPU baseline).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
package.  The product package never does.
"""
