#!/bin/sh
# build libtlk.so in-tree (prints the library path or the compiler error tail)
python -c "
from paper_2410_22254_b200.build import build
try: print(build())
except Exception as e: print(str(e)[-4000:]); raise SystemExit(1)"
