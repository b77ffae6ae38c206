python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
proj() { echo "== $*"; env "$@" timeout -s KILL 400 python scripts/scaling_projection.py 2>&1 | grep -E "worst"; }
proj B2_SLAB_BX=32
proj B2_SLAB_BX=64
proj B2_SLAB_BX=64 B2_SLAB_VEC=10
proj B2_SLAB_BX=32 B2_SLAB_VEC=10
proj B2_SLAB_BX=32 B2_MARCH_BY=16
