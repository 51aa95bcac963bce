"""TEST INFRASTRUCTURE ONLY (see abed_oracle.h): ctypes access to the C oracle
(liboracle.so) and to the reference implementation compiled in place
(_ref/libabed_ref*.so).  Imported only by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs."""
