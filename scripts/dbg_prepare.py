import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
from paper_2602_06991_b200 import api, synth
from paper_2602_06991_b200.types import RenderSettings, Pose
r = api.Renderer(0)
m = synth.random_scene(300, 8, 1); c = synth.test_camera(64, 48)
p = r.prepare_scene(m, Pose(), c, RenderSettings())
print('ok', len(p.src))
