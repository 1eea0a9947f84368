"""The one piece of the reference's sandbox service the reference test
fixtures use (conftest.demo_scene_256): the per-(scene, n) asset cache of
/root/reference/pkg/src/geofield/service.py:32-38, restated over this
package (TEST INFRASTRUCTURE; the service itself is out of scope)."""

from paper_1711_05017_b200.scenes import get_scene

_ASSET_CACHE = {}


def scene_assets(name, n=256):
    key = (name, n)
    if key not in _ASSET_CACHE:
        scene = get_scene(name)
        _ASSET_CACHE[key] = (scene, *scene.build_assets(n=n))
    return _ASSET_CACHE[key]
