"""A small run of every kernel family for compute-sanitizer (one tool per call): config 1 (fp64) on the
sweep + fix-up passes and the whole-grid path, and a 256^2 fp32 config-3 crop at K = 4.
    compute-sanitizer --tool memcheck python tools/sanitize_small.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from inputs import configs
    from paper_1609_07114_b200 import from_scene

    s = configs.make("cfg1")
    for whole in (False, True):
        sim = from_scene(s, device=0, whole_grid=whole)
        sim.record_energy(True)
        sim.step(40)
        sim.probe(); sim.energy(); sim.get_window()
        sim.close()
    s = configs.make("cfg3", n=256)
    sim = from_scene(s, device=0)
    sim.record_energy(True)
    sim.step(16)
    sim.probe(); sim.energy(); sim.get_window()
    print("steps_per_pass", sim.info().steps_per_pass)
    sim.close()
    print("sanitize_small: done")


if __name__ == "__main__":
    main()
