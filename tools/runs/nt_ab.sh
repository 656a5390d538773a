for lib in paper_2205_12721_b200/libtmop_b200.so vlibs/nt1/libtmop_b200.so; do echo "== $lib"; TMOP_LIB=$lib python tools/time_c2.py; done
