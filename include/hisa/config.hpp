// Forwarding header: the declarations the reference keeps in hisa/config.hpp live in hisa/api.hpp.
#pragma once
#include "hisa/api.hpp"
