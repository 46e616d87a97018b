mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_geometry.py -q -x --durations=4 > gpurun_out/geo2_test.log 2>&1; echo test=$?
tail -8 gpurun_out/geo2_test.log
python - <<'PY'
import time, sys
sys.path.insert(0, '.')
import paper_1703_08015_b200 as P
for phi in (0.2, 0.5, 0.8):
    t0 = time.time()
    g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(1024, 1024, 1024), sphere_diameter=40, target_porosity=phi, seed=7), device=0)
    print("1024^3 phi", phi, "->", round(P.porosity(g).phi, 4), "in", round(time.time() - t0, 2), "s")
PY
