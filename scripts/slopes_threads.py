import numpy as np, time, concurrent.futures as cf, os, sys
sys.path.insert(0, '.')
import paper_2404_14044_b200 as hp
from paper_2404_14044_b200 import pipeline
from paper_2404_14044_b200.geometry import radius_slopes
print(os.cpu_count(), len(os.sched_getaffinity(0)))
cam = hp.scene_camera(800, 800, fov_deg=40)
dirs, pix = hp.ray_grid(cam)
for _ in range(3):
    t=time.perf_counter(); a = radius_slopes(cam, pix, 0.0123); t1=time.perf_counter(); b = pipeline.host_slopes(cam, pix, 0.0123); t2=time.perf_counter()
    print(np.array_equal(a,b), (t1-t)*1e3, (t2-t1)*1e3)
