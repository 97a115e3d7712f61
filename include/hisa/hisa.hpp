// Forwarding header: the declarations the reference keeps in hisa/hisa.hpp live in hisa/api.hpp.
#pragma once
#include "hisa/api.hpp"
